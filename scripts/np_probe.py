import sys, time, statistics
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2210_03052_b200 as bt
from paper_2210_03052_b200 import harness, _lib
seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
w = bt.init_weights(cfg, 0)
xn = harness.gen_input(seqs, 768, 0)
x = bt.Tensor(xn)
for _ in range(3): bt.forward(w, seqs, x, cfg)
eng = bt.engine_for(w, cfg)
out = torch.empty((16*256, 768), dtype=torch.float32, pin_memory=True)
def t(fn, n=20):
    ts=[]
    for _ in range(n):
        torch.cuda.synchronize(); t0=time.perf_counter(); fn(); torch.cuda.synchronize(); ts.append(time.perf_counter()-t0)
    return statistics.median(ts)*1e3
print("pageable engine call", t(lambda: eng.forward_host_pageable(seqs, xn, out)))
xp = torch.from_numpy(xn).pin_memory()
print("pinned engine call", t(lambda: eng.forward_host_packed(seqs, xp, out)))
print("forward numpy", t(lambda: bt.forward(w, seqs, x, cfg)))
print("forward pinned", t(lambda: bt.forward(w, seqs, xp, cfg)))
print("torch.empty pinned", t(lambda: torch.empty((16*256, 768), dtype=torch.float32, pin_memory=True)))
print("Tensor(out.numpy())", t(lambda: bt.Tensor(out.numpy())))
