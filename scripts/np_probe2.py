"""Phase timing of the pageable-input host path (C2)."""
import sys, time, statistics, concurrent.futures as cf
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2210_03052_b200 as bt
from paper_2210_03052_b200 import harness, _lib
seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
w = bt.init_weights(cfg, 0)
xn = harness.gen_input(seqs, 768, 0)
eng = bt.engine_for(w, cfg)
out = torch.empty((16*256, 768), dtype=torch.float32, pin_memory=True)
eng.forward_host_pageable(seqs, xn, out)
graph, run, xp, yp, _, _ = eng._graph_entry(seqs, cfg, eng._cfg_c)
stage = eng._stage[(seqs.total, 768)]; sn = stage.array
L = np.asarray(seqs.lengths); st = np.concatenate([[0], np.cumsum(L)])
pool = eng._pool
bounds = eng.chunk_bounds(seqs.lengths, 8)
def cp(b0, b1):
    for b in range(b0, b1): sn[st[b]:st[b+1]] = xn[b*256: b*256+L[b]]
for rep in range(5):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for f in [pool.submit(cp, a, b) for a, b in bounds]: f.result()
    t1 = time.perf_counter()
    one = np.asarray([seqs.total], dtype=np.int32); _lib.call("bt_copy_rows", xp.data_ptr(), stage.ptr, one.ctypes.data, 1, seqs.total, 768 * 4, 1, _lib.stream_ptr())
    t2 = time.perf_counter()
    graph.replay()
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"stage {1e3*(t1-t0):.3f} copy_enq {1e3*(t2-t1):.3f} replay_enq {1e3*(t3-t2):.3f} sync {1e3*(t4-t3):.3f} total {1e3*(t4-t0):.3f}")
