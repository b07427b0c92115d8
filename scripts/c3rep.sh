# repeat bench runs and show per-step spread: bash scripts/c3rep.sh [configs]
cd $GRAFT_REPO_ROOT
for i in 1 2 3; do for c in ${@:-c3}; do BT_BENCH_STEPS_LOG=1 timeout -s KILL 300 python bench.py --config $c --no-cpu-baseline 2>&1 | grep -E "step|ms_per_step" | python -c "
import sys,json
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'): d=json.loads(l); print('$c ms/step', d['ms_per_step'], d['e2e']['value'], d['clocks'])
    else: print(l[:200])
"; done; done
