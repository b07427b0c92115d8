"""GEMM + bias + residual + LayerNorm cluster kernel alone at several shapes
(time per launch), for A/B of library variants via BT_LIB_PATH."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2210_03052_b200 import _lib
    _lib.require_device()
    for M, N, K in ((2458, 768, 768), (2458, 768, 3072), (4915, 1024, 1024), (4915, 1024, 4096), (1900, 1024, 4096)):
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = (torch.randn(N, K, device="cuda") / K ** 0.5).to(torch.bfloat16)
        r = torch.randn(M, N, device="cuda").to(torch.bfloat16)
        b, g, be = (torch.randn(N, device="cuda") for _ in range(3))
        y = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        go = lambda: _lib.call("bt_gemm_bias_residual_ln", a.data_ptr(), w.data_ptr(), b.data_ptr(), r.data_ptr(),  # noqa: E731
                               g.data_ptr(), be.data_ptr(), 1e-12, y.data_ptr(), M, N, K, _lib.stream_ptr())
        for _ in range(3):
            go()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            go()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        print(f"M={M} N={N} K={K}: {us:.2f} us  {2 * M * N * K / us / 1e6:.0f} TFLOP/s  checksum {y.float().abs().sum().item():.1f}")


if __name__ == "__main__":
    main()
