"""Per-CTA event timeline of one GEMM launch (globaltimer ns).

    python scripts/gemm_trace.py M N K EPI BN

Needs a trace build of the library (the trace points are compiled out otherwise):
    python -m paper_2210_03052_b200.build --variant scripts/ab/trace.so -D BT_TRACE_ON
    BT_LIB_PATH=scripts/ab/trace.so python scripts/gemm_trace.py ...
"""

import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.tensor import gemm_device

    _lib.require_device()
    M, N, K, epi, bn = map(int, sys.argv[1:6])
    if len(sys.argv) > 6:
        _lib.call("bt_debug_gemm_mode", int(sys.argv[6]))  # 3 = stream-K off, 4 = on
    A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
    W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
    bias = torch.randn(N, device="cuda") * 0.1
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    for _ in range(2000):  # warm: clocks up to their loaded level before the traced launch
        gemm_device(A, W, bias if epi else None, None, epi, out=C, bn=bn or None)
    buf = torch.zeros(148 * 64, dtype=torch.int64, device="cuda")
    _lib.call("bt_debug_gemm_trace", buf.data_ptr())
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    gemm_device(A, W, bias if epi else None, None, epi, out=C, bn=bn or None)
    ev1.record()
    torch.cuda.synchronize()
    _lib.call("bt_debug_gemm_trace", 0)
    print(f"shape {M}x{N}x{K} epi {epi} bn {bn}: event time {ev0.elapsed_time(ev1) * 1e3:.2f} us")
    t = buf.view(148, 64).cpu().numpy().astype(np.int64)
    used = t[:, 0] > 0
    t0 = t[used, 0].min()
    rel = lambda x: (x - t0) / 1e3  # noqa: E731
    print(f"CTAs traced: {used.sum()}  setup-done spread: {rel(t[used, 0]).min():.2f}..{rel(t[used, 0]).max():.2f} us")
    w = t[used, 62]
    f = t[used, 63]
    if (w > 0).any():
        print(f"griddep_wait returned: {rel(w[w > 0]).min():.2f}..{rel(w[w > 0]).max():.2f} us; first k-block landed: "
              f"median {np.median(rel(f[f > 0])):.2f} us")
    last = []
    for c in np.nonzero(used)[0][:6].tolist() + np.nonzero(used)[0][-3:].tolist():
        row = t[c]
        s = f"cta {c:3d}: setup {rel(row[0]):6.2f}"
        for it in range(9):
            mb, me, eb, ee = row[2 + 6 * it:6 + 6 * it]
            if mb == 0 and eb == 0:
                break
            s += f" | t{row[6 + 6 * it]}: mma {rel(mb):6.2f}-{rel(me):6.2f} epi {rel(eb):6.2f}-{rel(ee):6.2f}"
        print(s)
    ends = []
    for c in np.nonzero(used)[0]:
        row = t[c]
        e = max(row[5 + 6 * it] for it in range(9) if row[5 + 6 * it] > 0) if any(
            row[5 + 6 * it] > 0 for it in range(9)) else row[0]
        ends.append(rel(e))
    print(f"CTA finish times: min {min(ends):.2f} median {np.median(ends):.2f} max {max(ends):.2f} us")
    mm = []
    ep = []
    for c in np.nonzero(used)[0]:
        row = t[c]
        for it in range(9):
            mb, me, eb, ee = row[2 + 6 * it:6 + 6 * it]
            if mb > 0 and me > 0:
                mm.append((me - mb) / 1e3)
            if eb > 0 and ee > 0:
                ep.append((ee - eb) / 1e3)
    if mm:
        print(f"mainloop per tile (mma begin->last commit issue): median {np.median(mm):.2f} us, max {max(mm):.2f}")
    if ep:
        print(f"epilogue per tile: median {np.median(ep):.2f} us, max {max(ep):.2f}")


if __name__ == "__main__":
    main()
