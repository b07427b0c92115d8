"""Where forward()'s time goes for a pageable (numpy) input at C2: host
timestamps around each phase of BertEncoderB200.forward_host_pageable and
CUDA events on its three streams."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.encoder import _WcStage, engine_for

    seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    arr = harness.gen_input(seqs, 768, 0).astype(np.float32)
    for _ in range(3):
        bt.forward(w, seqs, bt.Tensor(arr), cfg)
    eng = engine_for(w, cfg)
    k, bs, mx, T = 768, 16, 256, seqs.total
    graph, run, xp, yp, _, _ = eng._graph_entry(seqs, cfg, eng._cfg_c)
    stage = _WcStage(T, k)
    sn = stage.array
    h2d, comp, d2h = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
    lengths_h = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
    starts = np.concatenate([[0], np.cumsum(lengths_h)])
    out = torch.empty((bs * mx, k), dtype=torch.float32, pin_memory=True)
    one = np.asarray([T], dtype=np.int32)
    import concurrent.futures as cf
    pool = cf.ThreadPoolExecutor(4)
    bounds = eng.chunk_bounds(seqs.lengths, 8)
    rows = {}
    for it in range(25):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
        t = [time.perf_counter()]

        def copy_group(b0, b1):
            for b in range(b0, b1):
                sn[starts[b]:starts[b + 1]] = arr[b * mx: b * mx + lengths_h[b]]

        for f in [pool.submit(copy_group, b0, b1) for b0, b1 in bounds]:
            f.result()
        t.append(time.perf_counter())  # staged
        with torch.cuda.stream(h2d):
            ev[0].record(h2d)
            _lib.call("bt_copy_rows", xp.data_ptr(), stage.ptr, one.ctypes.data, 1, T, k * 4, 1, _lib.stream_ptr())
            ev[1].record(h2d)
        comp.wait_stream(h2d)
        t.append(time.perf_counter())  # h2d enqueued
        with torch.cuda.stream(comp):
            graph.replay()
            ev[2].record(comp)
        t.append(time.perf_counter())  # graph enqueued
        eng._zero_padded_rows(out, seqs, k)
        t.append(time.perf_counter())  # host zeroing done
        d2h.wait_stream(comp)
        with torch.cuda.stream(d2h):
            ev[3].record(d2h)
            _lib.call("bt_copy_rows", out.data_ptr(), yp.data_ptr(), lengths_h.ctypes.data, bs, mx, k * 4, 0,
                      _lib.stream_ptr())
            ev[4].record(d2h)
        t.append(time.perf_counter())  # d2h enqueued
        d2h.synchronize()
        t.append(time.perf_counter())  # done
        if it >= 5:
            names = ["stage", "h2d_enq", "replay_enq", "zero", "d2h_enq", "sync"]
            for i, n in enumerate(names):
                rows.setdefault(n, []).append((t[i + 1] - t[i]) * 1e3)
            rows.setdefault("total", []).append((t[-1] - t[0]) * 1e3)
            rows.setdefault("dev_h2d", []).append(ev[0].elapsed_time(ev[1]))
            rows.setdefault("dev_h2d_to_graph_end", []).append(ev[1].elapsed_time(ev[2]))
            rows.setdefault("dev_graph_end_to_d2h_start", []).append(ev[2].elapsed_time(ev[3]))
            rows.setdefault("dev_d2h", []).append(ev[3].elapsed_time(ev[4]))
    for n, v in rows.items():
        print(f"{n:28s} median {statistics.median(v):.3f} ms")


if __name__ == "__main__":
    main()
