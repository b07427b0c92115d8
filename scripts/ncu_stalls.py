# Warp-stall samples per SASS line from an ncu --page source --csv --print-source sass export:
#   python scripts/ncu_stalls.py mha_c3_sass.csv [top_n]
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h:i for i,h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = collections.Counter()
per = []
for r in data:
    if len(r) < len(hdr): continue
    try: s = int(r[ix['Warp Stall Sampling (All Samples)']] or 0)
    except: continue
    per.append((s, r[ix['Address']], r[ix['Source']][:70], {c:int(r[ix[c]] or 0) for c in stall_cols}))
    for c in stall_cols: tot[c] += int(r[ix[c]] or 0)
S = sum(tot.values())
print("total samples", S)
for c,v in tot.most_common(12): print(f"  {c:28s} {v:7d} {100*v/S:5.1f}%")
per.sort(key=lambda x:-x[0])
for s,a,src,d in per[:int(sys.argv[2]) if len(sys.argv)>2 else 30]:
    top = sorted(d.items(), key=lambda x:-x[1])[:3]
    print(f"{s:6d} {100*s/S:5.1f}% {a} {src:70s} {' '.join(f'{k[6:]}={v}' for k,v in top)}")
