"""Per-CTA event timeline of one MHA launch (globaltimer ns).

    python scripts/mha_trace.py c2|c3

Needs a trace build of the library (the trace points are compiled out otherwise):
    python -m paper_2210_03052_b200.build --variant scripts/ab/trace.so -D BT_TRACE_ON
    BT_LIB_PATH=scripts/ab/trace.so python scripts/mha_trace.py ...
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.attention import mha_device
    from paper_2210_03052_b200.packing import plan_for_lengths

    _lib.require_device()
    bs, mx, H = {"c2": (16, 256, 12), "c3": (16, 512, 16), "c5": (2048, 512, 16)}[sys.argv[1]]
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    plan = plan_for_lengths(seqs)
    qkv = torch.randn(plan.valid_word_cnt, 3 * H * 64, device="cuda").to(torch.bfloat16)
    for _ in range(2000):  # warm: clocks up to their loaded level before the traced launch
        mha_device(qkv, plan, H, 64)
    nq = (mx + 127) // 128
    n = nq * H * bs
    if len(sys.argv) > 2 and sys.argv[2] == "list":
        return trace_list(torch, np, _lib, plan, qkv, seqs, bs, mx, H, n)
    if len(sys.argv) > 2 and sys.argv[2] == "seg":
        return trace_seg(torch, np, _lib, plan, qkv, bs, mx, H)
    buf = torch.zeros(n * 32, dtype=torch.int64, device="cuda")
    _lib.call("bt_debug_mha_trace", buf.data_ptr())
    mha_device(qkv, plan, H, 64)
    torch.cuda.synchronize()
    _lib.call("bt_debug_mha_trace", 0)
    t = buf.view(n, 32).cpu().numpy()
    used = t[:, 0] > 0
    t0 = t[used, 0].min()
    r = lambda x: (x - t0) / 1e3  # noqa: E731
    starts = r(t[used, 0])
    ends = r(t[used, 31])
    print(f"{sys.argv[1]}: CTAs active {used.sum()} of {n}; start spread {starts.min():.2f}..{starts.max():.2f} us;"
          f" end {ends.min():.2f}..{ends.max():.2f} us; per-CTA duration median {np.median(ends - starts):.2f} us")
    lens = seqs.lengths
    for c in np.nonzero(used)[0][:4].tolist() + np.nonzero(used)[0][-2:].tolist():
        row = t[c]
        qt, rest = c % nq, c // nq
        h, b = rest % H, rest // H
        s = f"cta q{qt} h{h} b{b} len {lens[b]}: start {r(row[0]):.2f} Q {r(row[1]):.2f} |"
        for i in range(7):
            if row[2 + 2 * i] == 0:
                break
            s += f" S{i} {r(row[2 + 2 * i]):.2f}-{r(row[3 + 2 * i]):.2f}"
        s += f" | O {r(row[30]):.2f} st {r(row[31]):.2f}"
        print(s)
    q_lat = t[used, 1] - t[used, 0]
    print(f"Q-load latency median {np.median(q_lat) / 1e3:.2f} us")
    s0 = t[used, 2] - t[used, 1]
    print(f"Q->S0 ready median {np.median(s0) / 1e3:.2f} us")
    soft = [(t[c, 3 + 2 * i] - t[c, 2 + 2 * i]) / 1e3 for c in np.nonzero(used)[0] for i in range(7)
            if t[c, 2 + 2 * i] > 0 and t[c, 3 + 2 * i] > 0]
    gaps = [(t[c, 2 + 2 * (i + 1)] - t[c, 3 + 2 * i]) / 1e3 for c in np.nonzero(used)[0] for i in range(6)
            if t[c, 2 + 2 * (i + 1)] > 0 and t[c, 3 + 2 * i] > 0]
    print(f"softmax per item median {np.median(soft):.2f} us; item-done -> next S ready median {np.median(gaps):.2f} us")
    for j in range(3):
        rows = [c for c in np.nonzero(used)[0] if t[c, 2 + 2 * j] > 0 and t[c, 19 + 4 * j] > 0]
        if not rows:
            break
        d = lambda a, b: np.median([(t[c, b] - t[c, a]) / 1e3 for c in rows])  # noqa: E731
        print(f"item {j} (n={len(rows)}): S ready->in regs {d(2 + 2 * j, 16 + 4 * j):.2f}  max {d(16 + 4 * j, 17 + 4 * j):.2f}"
              f"  wait PV {d(17 + 4 * j, 18 + 4 * j):.2f}  exps+store {d(18 + 4 * j, 19 + 4 * j):.2f}"
              f"  rescale+arrive {d(19 + 4 * j, 3 + 2 * j):.2f} us")
    fin = [(t[c, 31] - t[c, 30]) / 1e3 for c in np.nonzero(used)[0]]
    print(f"O ready -> stored median {np.median(fin):.2f} us")


def trace_list(torch, np, _lib, plan, qkv, seqs, bs, mx, H, n):
    """Balanced tile-list mode (bt_mha_varlen_sched, forced): per-CTA start,
    per-tile store times (slots 24..29), end."""
    T = plan.valid_word_cnt
    sched = torch.zeros(_lib.load().bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)
    mode = int(sys.argv[3]) if len(sys.argv) > 3 else 2

    def go():
        _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx, H,
                  64, 384, out.data_ptr(), T, _lib.stream_ptr())

    _lib.call("bt_debug_mha_list", mode, 0)
    for _ in range(2000):
        go()
    buf = torch.zeros(n * 32, dtype=torch.int64, device="cuda")
    _lib.call("bt_debug_mha_trace", buf.data_ptr())
    go()
    torch.cuda.synchronize()
    _lib.call("bt_debug_mha_trace", 0)
    _lib.call("bt_debug_mha_list", -1, 0)
    t = buf.view(n, 32).cpu().numpy()
    used = np.nonzero(t[:, 0] > 0)[0]
    t0 = t[used, 0].min()
    r = lambda x: (x - t0) / 1e3  # noqa: E731
    ends = r(t[used, 31])
    print(f"list mode {mode}: CTAs {len(used)}; start {r(t[used, 0]).min():.2f}..{r(t[used, 0]).max():.2f} us; "
          f"end {ends.min():.2f}..{ends.max():.2f} us (median {np.median(ends):.2f})")
    # slots 28, 29: tiles 1 and 2 stored
    k = 1 + (t[used, 28] > 0) + (t[used, 29] > 0)
    for nt in sorted(set(k.tolist())):
        cs = used[k == nt]
        print(f"  {len(cs)} CTAs with {nt}{'+' if nt == 3 else ''} tiles: end median {np.median(r(t[cs, 31])):.2f} us, "
              f"tile 1 {np.median((t[cs, 28] - t[cs, 0]) / 1e3) if nt > 1 else 0:.2f} us after start")
    for c in list(used[:3]) + list(used[-3:]):
        print(f"  cta {c}: start {r(t[c, 0]):.2f} Q {r(t[c, 1]):.2f} S0 {r(t[c, 2]):.2f} tiles 1,2 stored "
              + " ".join(f"{r(x):.2f}" for x in t[c, 28:30] if x > 0) + f" end {r(t[c, 31]):.2f}")

def trace_seg(torch, np, _lib, plan, qkv, bs, mx, H):
    """Segment kernel (forced): per-CTA start, S-ready / softmax-done per key
    block, output stored."""
    T = plan.valid_word_cnt
    sched = torch.zeros(_lib.load().bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)

    def go():
        _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx, H,
                  64, 384, out.data_ptr(), T, _lib.stream_ptr())

    _lib.call("bt_debug_mha_seg", 2)
    for _ in range(2000):
        go()
    n = bs * ((mx + 127) // 128) * H  # grid (H, bs * ceil(mx / 128)); CTAs past the item list exit
    buf = torch.zeros(n * 32, dtype=torch.int64, device="cuda")
    _lib.call("bt_debug_mha_trace", buf.data_ptr())
    go()
    torch.cuda.synchronize()
    _lib.call("bt_debug_mha_trace", 0)
    _lib.call("bt_debug_mha_seg", -1)
    t = buf.view(n, 32).cpu().numpy()
    used = np.nonzero(t[:, 0] > 0)[0]
    t0 = t[used, 0].min()
    r = lambda x: (x - t0) / 1e3  # noqa: E731
    ends = r(t[used, 31])
    nblk = np.array([sum(1 for i in range(7) if t[c, 2 + 2 * i] > 0) for c in used])
    print(f"segment kernel: CTAs {len(used)} of {n}; start {r(t[used, 0]).min():.2f}..{r(t[used, 0]).max():.2f} us; "
          f"end {ends.min():.2f}..{ends.max():.2f} (median {np.median(ends):.2f}); key blocks per CTA "
          f"{dict(zip(*np.unique(nblk, return_counts=True)))}")
    for k in sorted(set(nblk.tolist())):
        cs = used[nblk == k]
        print(f"  {len(cs)} CTAs with {k} blocks: duration median {np.median((t[cs, 31] - t[cs, 0]) / 1e3):.2f} us")
    for c in list(used[:2]) + list(used[-2:]):
        row = t[c]
        s = f"  cta {c}: start {r(row[0]):.2f} Q {r(row[1]):.2f} |"
        for i in range(7):
            if row[2 + 2 * i] == 0:
                break
            s += f" S{i} {r(row[2 + 2 * i]):.2f}-{r(row[3 + 2 * i]):.2f}"
        print(s + f" | O {r(row[30]):.2f} st {r(row[31]):.2f}")


if __name__ == "__main__":
    main()
