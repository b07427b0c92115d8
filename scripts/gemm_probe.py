"""Where a small-M GEMM's time goes: each C2 / C3 layer GEMM timed (CUDA
events over back-to-back launches, L2-warm) with the debug probes of
bt_debug_gemm_mode: 0 normal, 1 no MMAs (TMA feed alone), 2 no TMA loads
(MMA + epilogue), 6 no output store, 7 no TMEM loads, 8 TMEM loads only.

    python scripts/gemm_probe.py [c2|c3] [bn ...]
"""

import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

SHAPES = {
    "c2": [("qkv", 2458, 2304, 768, 1), ("attn_out", 2458, 768, 768, 0), ("ffn1", 2458, 3072, 768, 2),
           ("ffn2", 2458, 768, 3072, 0)],
    "c3": [("qkv", 4917, 3072, 1024, 1), ("attn_out", 4917, 1024, 1024, 0), ("ffn1", 4917, 4096, 1024, 2),
           ("ffn2", 4917, 1024, 4096, 0)],
}


def main():
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.tensor import gemm_device

    _lib.require_device()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
    bns = [int(b) for b in sys.argv[2:]] or [0]
    for name, M, N, K, epi in SHAPES[cfg]:
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
        bias = torch.randn(N, device="cuda") * 0.1
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        for bn in bns:
            if bn and (N % 64 or 4 * (-(-N // abs(bn)) * abs(bn) - N) > N):
                continue  # the library's partial-last-tile rule
            row = []
            for mode in (0, 1, 2, 6, 7, 8):
                _lib.call("bt_debug_gemm_mode", mode)
                f = lambda: gemm_device(A, W, bias if epi else None, None, epi, out=C, bn=bn or None)  # noqa
                for _ in range(20):
                    f()
                torch.cuda.synchronize()
                best = 1e9
                for _ in range(5):
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    torch.cuda._sleep(2_000_000)
                    e0.record()
                    for _ in range(10):
                        f()
                    e1.record()
                    torch.cuda.synchronize()
                    best = min(best, e0.elapsed_time(e1) * 100)
                row.append(best)
            _lib.call("bt_debug_gemm_mode", 0)
            fl = 2 * M * N * K
            print(f"{cfg} {name:9s} {M}x{N}x{K} epi {epi} bn {bn:5d}: normal {row[0]:6.2f} us ({fl / row[0] / 1e6:6.1f} "
                  f"TF/s) | feed-only {row[1]:6.2f} | mma+epi {row[2]:6.2f} | no-store {row[3]:6.2f} | "
                  f"no-tmem-ld {row[4]:6.2f} | tmem-ld-only {row[5]:6.2f}", flush=True)


if __name__ == "__main__":
    main()
