"""LayerNorm alone at C5 size (T = 629,146, k = 1024), back to back on a cool
GPU: GB/s against the bench's in-step figure."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.fusion import ln_device
    _lib.require_device()
    T, k = 629146, 1024
    x = torch.randn(T, k, device="cuda").to(torch.bfloat16)
    r = torch.randn(T, k, device="cuda").to(torch.bfloat16)
    b, g, be = (torch.randn(k, device="cuda") for _ in range(3))
    out = torch.empty_like(x)
    for n in (1, 5, 20):
        for _ in range(2):
            ln_device(x, r, b, g, be, 1e-12, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(n):
            ln_device(x, r, b, g, be, 1e-12, out=out)
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        print(f"{n} reps: {us:.1f} us/launch, {3 * T * k * 2 / us / 1e3:.0f} GB/s")


if __name__ == "__main__":
    main()
