"""forward_stream with reference-style numpy inputs at C2: wall time per
batch over a 20-batch stream (host inputs pageable)."""
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
    batches = [(seqs, bt.Tensor(harness.gen_input(seqs, 768, i))) for i in range(20)]
    bt.forward_stream(w, batches[:3], cfg)
    ts = []
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        bt.forward_stream(w, batches, cfg)
        ts.append((time.perf_counter() - t0) * 1e3 / len(batches))
    print(f"forward_stream(numpy) {statistics.median(ts):.3f} ms per batch")




if __name__ == "__main__":
    main()
