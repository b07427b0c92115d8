"""Every GEMM tile width (incl. partial last N tiles and the narrow-chunk
stores of 112/176/224/240-wide tiles) and epilogue once, plus a small
BERT-large-width forward (four-CTA MHA, GEMM + LN), for compute-sanitizer:

    compute-sanitizer --tool memcheck python scripts/sanitize_gemm.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200.tensor import gemm_device

    bt._lib.require_device()
    for M, N, K in ((300, 1024, 256), (129, 768, 128), (257, 2304, 64)):
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        w = torch.randn(N, K, device="cuda").to(torch.bfloat16)
        bias = torch.randn(N, device="cuda")
        res = torch.randn(M, N, device="cuda").to(torch.bfloat16)
        for bn in (64, 128, 192, 256, -112, -128, -176, -192, -224, -240, -256):
            for epi in (0, 1, 2, 3):
                gemm_device(a, w, bias if epi else None, res if epi == 3 else None, epi, bn=bn)
        torch.cuda.synchronize()
    lens = [512, 300, 129, 1, 77, 450, 256, 64]
    cfg = bt.ModelConfig(layers=2, head_num=16, head_size=64, max_seq_len=512, batch_size=len(lens),
                         flags=bt.OptFlags.all_on())
    x = torch.randn(len(lens) * 512, 1024, device="cuda")
    y = bt.forward(bt.init_weights(cfg, 0), bt.SeqLengths.of(lens, 512), x, cfg)
    torch.cuda.synchronize()
    print("sanitize gemm/forward done", bool(torch.isfinite(y).all().item()))


if __name__ == "__main__":
    main()
