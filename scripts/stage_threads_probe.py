import sys, time, statistics
sys.path.insert(0, '.')
import numpy as np
import concurrent.futures as cf
import torch
import paper_2210_03052_b200 as bt
from paper_2210_03052_b200 import harness
from paper_2210_03052_b200.encoder import _WcStage
seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
x = harness.gen_input(seqs, 768, 0).astype(np.float32)
L = np.asarray(seqs.lengths); starts = np.concatenate([[0], np.cumsum(L)]); T = int(starts[-1])
for kind in ("wc", "pinned"):
    if kind == "wc":
        st = _WcStage(T, 768); sn = st.array
    else:
        pt = torch.empty((T, 768), dtype=torch.float32, pin_memory=True); sn = pt.numpy()
    for nt in (1, 2, 4, 8, 16):
        pool = cf.ThreadPoolExecutor(nt)
        bounds = np.array_split(np.arange(16), nt)
        def grp(bb):
            for b in bb:
                sn[starts[b]:starts[b+1]] = x[b*256:b*256+L[b]]
        ts = []
        for _ in range(30):
            t0 = time.perf_counter()
            for f in [pool.submit(grp, bb) for bb in bounds if len(bb)]: f.result()
            ts.append(time.perf_counter() - t0)
        print(kind, nt, "threads: median %.3f ms" % (statistics.median(ts[5:]) * 1e3), flush=True)
        pool.shutdown()
cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
w = bt.init_weights(cfg, 0)
X = bt.Tensor(x)
for _ in range(5): y = bt.forward(w, seqs, X, cfg)
ts = []
for _ in range(30):
    t0 = time.perf_counter(); y = bt.forward(w, seqs, X, cfg); ts.append(time.perf_counter() - t0)
print("forward(numpy) median %.3f ms" % (statistics.median(ts) * 1e3))
import os; print("cpus", len(os.sched_getaffinity(0)))
