import sys, time, numpy as np, concurrent.futures as cf
sys.path.insert(0, '/root/repo')
import torch
from paper_2210_03052_b200 import harness
seqs = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
x = harness.gen_input(seqs, 768, 0)
L = np.asarray(seqs.lengths); st = np.concatenate([[0], np.cumsum(L)])
stage = torch.empty((seqs.total, 768), dtype=torch.float32, pin_memory=True); sn = stage.numpy()
def cp(b0, b1):
    for b in range(b0, b1): sn[st[b]:st[b+1]] = x[b*256: b*256+L[b]]
for name, fn in [("seq", lambda: cp(0, 16))]:
    for _ in range(3): fn()
    t=time.perf_counter(); [fn() for _ in range(20)]; print(name, (time.perf_counter()-t)/20*1e3, "ms")
for w in (2, 4, 8):
    pool = cf.ThreadPoolExecutor(w)
    bounds = [(i*16//8, (i+1)*16//8) for i in range(8)]
    def par():
        fs=[pool.submit(cp,a,b) for a,b in bounds]; [f.result() for f in fs]
    for _ in range(3): par()
    t=time.perf_counter(); [par() for _ in range(20)]; print("pool", w, (time.perf_counter()-t)/20*1e3, "ms")
t=time.perf_counter(); [np.copyto(np.empty_like(x), x) for _ in range(10)]; print("full 12.6MB copy to fresh", (time.perf_counter()-t)/10*1e3)
y=np.empty_like(x); t=time.perf_counter(); [np.copyto(y, x) for _ in range(10)]; print("full 12.6MB copy warm", (time.perf_counter()-t)/10*1e3)
import os; print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
