"""Where does the end-to-end forward() time go?  Host timestamps + CUDA events."""

import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import _lib, harness

    seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    x = torch.from_numpy(harness.gen_input(seqs, 768, 0)).pin_memory()
    for _ in range(5):
        y = bt.forward(w, seqs, x, cfg)
    torch.cuda.synchronize()
    eng = bt.engine_for(w, cfg)
    T, bs, mx, k = seqs.total, 16, 256, 768
    out = torch.empty((bs * mx, k), dtype=torch.float32, pin_memory=True)
    graph, run, xp, yp = eng._graph_entry(seqs, cfg, eng._cfg_c)[:4]
    lengths_h = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
    lp = lengths_h.ctypes.data
    s = _lib.stream_ptr()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ev[0].record()
        _lib.call("bt_copy_rows", xp.data_ptr(), x.data_ptr(), lp, bs, mx, k * 4, 1, s)
        t1 = time.perf_counter()
        ev[1].record()
        graph.replay()
        t2 = time.perf_counter()
        ev[2].record()
        _lib.call("bt_copy_rows", out.data_ptr(), yp.data_ptr(), lp, bs, mx, k * 4, 0, s)
        ev[3].record()
        t3 = time.perf_counter()
        o = out.numpy().reshape(bs, mx, k)
        for b, n in enumerate(seqs.lengths):
            if n < mx:
                o[b, n:] = 0.0
        t4 = time.perf_counter()
        torch.cuda.current_stream().synchronize()
        t5 = time.perf_counter()
        print(f"host: h2d-enq {1e3*(t1-t0):.3f} replay-enq {1e3*(t2-t1):.3f} d2h-enq {1e3*(t3-t2):.3f} "
              f"zero {1e3*(t4-t3):.3f} sync {1e3*(t5-t4):.3f} total {1e3*(t5-t0):.3f} ms | gpu: h2d "
              f"{ev[0].elapsed_time(ev[1]):.3f} graph {ev[1].elapsed_time(ev[2]):.3f} d2h {ev[2].elapsed_time(ev[3]):.3f}")
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        y = bt.forward(w, seqs, x, cfg)
        t1 = time.perf_counter()
        print(f"forward() {1e3*(t1-t0):.3f} ms")
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        y = bt.forward(w, seqs, x, cfg)
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)


if __name__ == "__main__":
    main()
