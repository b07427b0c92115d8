"""Host profile of forward() with a pageable (numpy Tensor) input at C2."""
import cProfile
import pstats
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import harness

    seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    x = bt.Tensor(harness.gen_input(seqs, 768, 0))
    for _ in range(5):
        y = bt.forward(w, seqs, x, cfg)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        t0 = time.perf_counter()
        y = bt.forward(w, seqs, x, cfg)
        ts.append(time.perf_counter() - t0)
    print(f"forward(numpy) median {statistics.median(ts) * 1e3:.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        y = bt.forward(w, seqs, x, cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(14)


if __name__ == "__main__":
    main()
