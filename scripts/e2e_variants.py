"""C2 e2e variants: raw PCIe copy rates and the public forward on host
buffers by (A) per-sequence DMA around the cached graph, (B) zero-copy
(the prologue reads the pinned input, the last LayerNorm writes the pinned
output), (C) zero-copy input + DMA output.

    python scripts/e2e_variants.py
"""
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

    bs, mx, k = 16, 256, 768
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config("bert_base", bs, mx, bt.OptFlags.all_on())
    w = bt.init_weights(cfg, 0)
    xh = torch.from_numpy(harness.gen_input(seqs, k, 0)).pin_memory()
    oh = torch.empty((bs * mx, k), dtype=torch.float32).pin_memory()
    T = seqs.total
    big = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream()

    def dev_time(fn, n=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(n):
            fn()
        b.record(s)
        torch.cuda.synchronize()
        return a.elapsed_time(b) / n * 1e3

    nb = T * k * 4
    dpk = torch.empty((T, k), dtype=torch.float32, device="cuda")
    hpk = torch.empty((T, k), dtype=torch.float32).pin_memory()
    lh = np.ascontiguousarray(np.asarray(seqs.lengths, dtype=np.int32))
    print(f"one {nb / 1e6:.2f} MB H2D copy: {dev_time(lambda: dpk.copy_(hpk, non_blocking=True)):.1f} us")
    print(f"one {nb / 1e6:.2f} MB D2H copy: {dev_time(lambda: hpk.copy_(dpk, non_blocking=True)):.1f} us")
    print(f"per-sequence H2D (bt_copy_rows): {dev_time(lambda: _lib.call('bt_copy_rows', dpk.data_ptr(), xh.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 1, _lib.stream_ptr())):.1f} us")
    print(f"per-sequence D2H (bt_copy_rows): {dev_time(lambda: _lib.call('bt_copy_rows', oh.data_ptr(), dpk.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 0, _lib.stream_ptr())):.1f} us")

    eng = bt.engine_for(w, cfg)
    lengths_dev = torch.tensor(seqs.lengths, dtype=torch.int32, device="cuda")
    od = torch.empty((bs * mx, k), dtype=torch.float32, device="cuda")
    xd = xh.cuda()

    def wall(fn, n=30):
        for _ in range(5):
            fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(n):
            big.zero_()
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        return statistics.median(ts) * 1e3

    def a():
        eng.forward_host_packed(seqs, xh, oh)

    def b_zero_copy():
        eng.forward_ptrs(lengths_dev.data_ptr(), bs, T, xh.data_ptr(), oh.data_ptr())

    def c_zc_in():
        eng.forward_ptrs(lengths_dev.data_ptr(), bs, T, xh.data_ptr(), od.data_ptr())
        _lib.call("bt_copy_rows", oh.data_ptr(), od.data_ptr(), lh.ctypes.data, bs, mx, k * 4, 0, _lib.stream_ptr())

    def d_device():
        eng.forward_ptrs(lengths_dev.data_ptr(), bs, T, xd.data_ptr(), od.data_ptr())

    ref = None
    for name, fn in (("A per-seq DMA + graph", a), ("B zero-copy in+out (eager)", b_zero_copy),
                     ("C zero-copy in + DMA out (eager)", c_zc_in), ("D device buffers (eager)", d_device)):
        t = wall(fn)
        torch.cuda.synchronize()
        res = (od.cpu() if name.startswith("D") else oh.clone())
        if ref is None:
            ref = res
        print(f"{name}: {t:.3f} ms per forward (wall, synchronised); == A: {torch.equal(ref, res)}", flush=True)
    print(f"device time of D: {dev_time(d_device):.1f} us; B: {dev_time(b_zero_copy):.1f} us; C: {dev_time(c_zc_in):.1f} us")


if __name__ == "__main__":
    main()
