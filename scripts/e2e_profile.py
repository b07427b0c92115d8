"""Host time of the public forward() on pinned host buffers (C2): cProfile
of 50 calls plus wall time with and without the output allocation."""
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
    x = torch.from_numpy(harness.gen_input(seqs, 768, 0)).pin_memory()
    y = None
    for _ in range(5):
        y = bt.forward(w, seqs, x, cfg)
    torch.cuda.synchronize()

    def wall(fn, n=40):
        ts = []
        for _ in range(n):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3

    def fwd():
        global _keep
        _keep = bt.forward(w, seqs, x, cfg)

    eng = bt.engine_for(w, cfg)
    out = torch.empty((16 * 256, 768), dtype=torch.float32, pin_memory=True)
    print(f"forward() median {wall(fwd):.3f} ms")
    print(f"engine.forward_host_packed (preallocated out) median {wall(lambda: eng.forward_host_packed(seqs, x, out)):.3f} ms")
    print(f"torch.empty pinned 12.6 MB median {wall(lambda: torch.empty((16 * 256, 768), dtype=torch.float32, pin_memory=True)):.3f} ms")
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(50):
        fwd()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
