"""Is the GEMM's TMA feed limited per SM or chip-wide?  Time the pure-feed
mode (MMAs skipped) with few vs all SMs active, 1-CTA 128x128 tiles."""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.tensor import gemm_device

    _lib.require_device()
    K = 12288
    for mode in (1, 0):
        _lib.call("bt_debug_gemm_mode", mode)
        _lib.call("bt_debug_gemm_mode", 3)  # no stream-K
        for ctas, bn in ((8, 128), (16, 128), (37, 128), (74, 128), (148, 128), (148, 256), (74, -256)):
            rows = 128 * ctas if bn > 0 else 256 * ctas
            n = abs(bn) if bn > 0 else 256
            A = torch.randn(rows, K, device="cuda").to(torch.bfloat16)
            W = torch.randn(n, K, device="cuda").to(torch.bfloat16)
            C = torch.empty(rows, n, device="cuda", dtype=torch.bfloat16)
            for _ in range(2):
                gemm_device(A, W, out=C, bn=bn)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            for _ in range(5):
                gemm_device(A, W, out=C, bn=bn)
            e1.record()
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / 5
            per_cta_bytes = (128 + (n if bn > 0 else n // 2)) * K * 2
            total = per_cta_bytes * (ctas if bn > 0 else 2 * ctas)
            sm_clk = 1.965e3  # MHz
            print(f"mode {mode} ctas {ctas if bn > 0 else 2 * ctas:4d} tile {bn:5d}: {us:8.1f} us  "
                  f"per-SM {per_cta_bytes / (us * sm_clk):6.1f} B/clk  chip {total / us / 1e3:7.2f} TB/s")
    _lib.call("bt_debug_gemm_mode", 0)
    _lib.call("bt_debug_gemm_mode", 5)


if __name__ == "__main__":
    main()
