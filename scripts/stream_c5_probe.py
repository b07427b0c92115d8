"""Where forward_stream's time goes at C5: per-batch graph time (events on the
compute stream) and the wall time of the whole stream vs K x per-call."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import harness
    bs, mx, k = 2048, 512, 1024
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    cfg = bt.ModelConfig(layers=24, head_num=16, head_size=64, max_seq_len=mx, batch_size=bs, flags=bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    xh = harness.gen_input(seqs, k, 0)
    xs = [torch.from_numpy(xh).pin_memory(), torch.from_numpy(xh.copy()).pin_memory()]
    K = 4
    ys = bt.forward_stream(w, [(seqs, xs[i % 2]) for i in range(K)], cfg)
    ys = None
    torch.cuda.synchronize()
    eng = bt.engine_for(w, cfg)
    # instrument: wrap graph replays with events
    import paper_2210_03052_b200.encoder as enc
    evs = []
    orig = torch.cuda.CUDAGraph.replay

    def rep(self):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        orig(self)
        b.record()
        evs.append((a, b))
    torch.cuda.CUDAGraph.replay = rep
    t0 = time.perf_counter()
    ys = bt.forward_stream(w, [(seqs, xs[i % 2]) for i in range(K)], cfg)
    t1 = time.perf_counter()
    torch.cuda.CUDAGraph.replay = orig
    print(f"stream of {K}: {1e3 * (t1 - t0) / K:.1f} ms per batch; graph times "
          + " ".join(f"{a.elapsed_time(b):.1f}" for a, b in evs)
          + "; gaps " + " ".join(f"{evs[i][1].elapsed_time(evs[i + 1][0]):.1f}" for i in range(len(evs) - 1)))
    t0 = time.perf_counter()
    for i in range(K):
        y = bt.forward(w, seqs, xs[i % 2], cfg)
    t1 = time.perf_counter()
    print(f"{K} calls: {1e3 * (t1 - t0) / K:.1f} ms per batch")


if __name__ == "__main__":
    main()
