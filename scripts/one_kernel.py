"""Launch one kernel configuration a few times (ncu target).

    python scripts/one_kernel.py gemm M N K EPI BN
    python scripts/one_kernel.py mha c2|c3
    python scripts/one_kernel.py ln T K
"""

import math
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.packing import plan_for_lengths

    _lib.require_device()
    kind = sys.argv[1]
    if kind == "gemm":
        from paper_2210_03052_b200.tensor import gemm_device

        M, N, K, epi, bn = map(int, sys.argv[2:7])
        A = (torch.randn(M, K, device="cuda") * 0.5).to(torch.bfloat16)
        W = (torch.randn(N, K, device="cuda") / math.sqrt(K)).to(torch.bfloat16)
        bias = torch.randn(N, device="cuda") * 0.1
        for _ in range(8):
            gemm_device(A, W, bias if epi else None, None, epi, bn=bn if bn else None)
    elif kind == "mha":
        from paper_2210_03052_b200.attention import mha_device

        cfgs = {"c2": (16, 256, 12), "c3": (16, 512, 16)}
        bs, mx, H = cfgs[sys.argv[2]]
        seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
        plan = plan_for_lengths(seqs)
        qkv = torch.randn(plan.valid_word_cnt, 3 * H * 64, device="cuda").to(torch.bfloat16)
        for _ in range(8):
            mha_device(qkv, plan, H, 64)
    elif kind == "ln":
        from paper_2210_03052_b200.fusion import ln_device

        T, K = int(sys.argv[2]), int(sys.argv[3])
        x = torch.randn(T, K, device="cuda").to(torch.bfloat16)
        g = torch.ones(K, device="cuda")
        for _ in range(3):
            ln_device(x, x, g, g, g, 1e-12)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
