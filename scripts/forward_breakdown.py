"""Per-kernel device time INSIDE a real encoder forward (events recorded by
the library between its launches; bt_debug_forward_events).

    python scripts/forward_breakdown.py [--config c2] [--reps 20]

Events between kernels cut the programmatic-dependent-launch overlap, so the
sum is a little above the graph-replayed step time; shares are what matter.
"""

import argparse
import ctypes as C
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    import numpy as np
    import torch

    import bench
    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import _lib, harness

    desc, heads, layers, bs, mx, _ = bench.WORKLOADS[a.config]
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    cfg = bt.ModelConfig(layers=layers, head_num=heads, head_size=64, max_seq_len=mx, batch_size=bs,
                         flags=bt.OptFlags.all_on())
    eng = bt.BertEncoderB200(bt.init_weights(cfg, 0), cfg)
    x = torch.from_numpy(harness.gen_input(seqs, heads * 64, 0)).cuda()
    lengths = torch.tensor(seqs.lengths, dtype=torch.int32, device="cuda")
    out = torch.empty_like(x)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        eng.forward_device(lengths, bs, seqs.total, x, out)
    n = 3 + 7 * layers
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
    for e in evs:
        e.record()
    torch.cuda.synchronize()
    handles = (C.c_void_p * n)(*[e.cuda_event for e in evs])
    names = ["qkv", "mha", "attn_out", "ln0", "ffn1", "ffn2", "ln1"]
    acc = np.zeros(n - 1)
    for _ in range(a.reps):
        flush.zero_()
        _lib.call("bt_debug_forward_events", handles, n)
        eng.forward_device(lengths, bs, seqs.total, x, out)
        _lib.call("bt_debug_forward_events", None, 0)
        torch.cuda.synchronize()
        acc += np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(n - 1)])
    acc = acc * 1e3 / a.reps  # us
    per = {"plan+pack": acc[0], "unpack": acc[-1]}
    for j, nm in enumerate(names):
        per[nm] = float(np.mean([acc[1 + 7 * li + j] for li in range(layers)]))
    tot = acc.sum()
    print(f"{desc}: forward {tot:.1f} us (events between launches)")
    for k, v in per.items():
        mult = 1 if k in ("plan+pack", "unpack") else layers
        print(f"  {k:10s} {v:8.2f} us x{mult:<3d} share {v * mult / tot:.3f}")


if __name__ == "__main__":
    main()
