"""H2D DMA rate of a 7.5 MB host buffer (C2's valid input rows) by how the
host buffer was last touched: write-combined (bt_host_alloc) vs cached
page-locked memory, just written by the CPU or not."""
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.encoder import _WcStage

    T, k = 2458, 768
    src = np.random.default_rng(0).standard_normal((T, k)).astype(np.float32)
    dev = torch.empty((T, k), dtype=torch.float32, device="cuda")
    wc = _WcStage(T, k)
    pin = torch.empty((T, k), dtype=torch.float32, pin_memory=True)
    pn = pin.numpy()
    s = torch.cuda.Stream()
    one = np.asarray([T], dtype=np.int32)

    def dma(ptr):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record(s)
            _lib.call("bt_copy_rows", dev.data_ptr(), ptr, one.ctypes.data, 1, T, k * 4, 1, _lib.stream_ptr())
            b.record(s)
        s.synchronize()
        return a.elapsed_time(b)

    import concurrent.futures as cf
    pool = cf.ThreadPoolExecutor(4)
    q = np.linspace(0, T, 9).astype(int)

    def pool_write(arr):
        def part(i):
            arr[q[i]:q[i + 1]] = src[q[i]:q[i + 1]]
        for f in [pool.submit(part, i) for i in range(8)]:
            f.result()

    cases = {
        "wc_after_pool_write": (lambda: pool_write(wc.array), wc.ptr),
        "pinned_after_pool_write": (lambda: pool_write(pn), pin.data_ptr()),
        "wc_after_write": (lambda: wc.array.__setitem__(slice(None), src), wc.ptr),
        "wc_no_write": (lambda: None, wc.ptr),
        "pinned_after_write": (lambda: pn.__setitem__(slice(None), src), pin.data_ptr()),
        "pinned_no_write": (lambda: None, pin.data_ptr()),
    }
    for name, (touch, ptr) in cases.items():
        ts = []
        for i in range(25):
            touch()
            ts.append(dma(ptr))
        ms = statistics.median(ts[5:])
        print(f"{name:22s} {ms:.3f} ms  {T * k * 4 / ms / 1e6:.1f} GB/s", flush=True)
    # pipelined: write 8 chunks, DMA each right after its write
    bounds = np.linspace(0, T, 9).astype(int)
    for name, arr, base in (("wc_pipelined8", wc.array, wc.ptr), ("pinned_pipelined8", pn, pin.data_ptr())):
        ts = []
        for i in range(25):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for c in range(8):
                r0, r1 = bounds[c], bounds[c + 1]
                arr[r0:r1] = src[r0:r1]
                n = np.asarray([r1 - r0], dtype=np.int32)
                with torch.cuda.stream(s):
                    _lib.call("bt_copy_rows", int(dev.data_ptr() + r0 * k * 4), int(base + r0 * k * 4), n.ctypes.data, 1,
                              int(r1 - r0), k * 4, 1, _lib.stream_ptr())
            s.synchronize()
            ts.append((time.perf_counter() - t0) * 1e3)
        print(f"{name:22s} {statistics.median(ts[5:]):.3f} ms host+DMA", flush=True)
    # pageable source straight to the device (driver staging)
    ts = []
    for i in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            _lib.call("bt_copy_rows", dev.data_ptr(), src.ctypes.data, one.ctypes.data, 1, T, k * 4, 1,
                      _lib.stream_ptr())
        s.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{'pageable_direct':22s} {statistics.median(ts[5:]):.3f} ms host wall", flush=True)
    ts = []
    for i in range(25):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        dev.copy_(torch.from_numpy(src), non_blocking=False)
        torch.cuda.synchronize()
        ts.append((time.perf_counter() - t0) * 1e3)
    print(f"{'torch_pageable_copy':22s} {statistics.median(ts[5:]):.3f} ms host wall", flush=True)


if __name__ == "__main__":
    main()
