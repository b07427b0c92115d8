"""Per-sequence PCIe copies (C2 valid rows, 16 sequences) spread over 1, 2, 4
streams: does overlapping the per-copy setup on several copy engines recover
the single-copy rate?"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib, harness

    bs, mx, k = 16, 256, 768
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    T = seqs.total
    xh = torch.from_numpy(harness.gen_input(seqs, k, 0)).pin_memory()
    oh = torch.empty((bs * mx, k), dtype=torch.float32).pin_memory()
    dpk = torch.empty((T, k), dtype=torch.float32, device="cuda")
    lens = list(seqs.lengths)
    starts = np.concatenate([[0], np.cumsum(lens)])
    main_s = torch.cuda.current_stream()
    pools = {n: [torch.cuda.Stream() for _ in range(n)] for n in (1, 2, 4, 8)}

    def run(n, to_dev):
        ss = pools[n]
        evs = []
        for st in ss:
            st.wait_stream(main_s)
        for b in range(bs):
            st = ss[b % n]
            with torch.cuda.stream(st):
                if to_dev:
                    dpk[starts[b]:starts[b + 1]].copy_(xh[b * mx: b * mx + lens[b]], non_blocking=True)
                else:
                    oh[b * mx: b * mx + lens[b]].copy_(dpk[starts[b]:starts[b + 1]], non_blocking=True)
        for st in ss:
            main_s.wait_stream(st)

    for to_dev in (True, False):
        for n in (1, 2, 4, 8):
            for _ in range(3):
                run(n, to_dev)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(20):
                run(n, to_dev)
            b.record()
            torch.cuda.synchronize()
            us = a.elapsed_time(b) / 20 * 1e3
            print(f"{'H2D' if to_dev else 'D2H'} per-sequence over {n} streams: {us:.1f} us "
                  f"({T * k * 4 / us / 1e3:.1f} GB/s)", flush=True)
    # both directions at once (full duplex)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s2 = torch.cuda.Stream()
    hpk = torch.empty((T, k), dtype=torch.float32).pin_memory()
    d2 = torch.empty((T, k), dtype=torch.float32, device="cuda")
    a.record()
    for _ in range(20):
        s2.wait_stream(main_s)
        dpk.copy_(hpk, non_blocking=True)
        with torch.cuda.stream(s2):
            hpk.copy_(d2, non_blocking=True)
        main_s.wait_stream(s2)
    b.record()
    torch.cuda.synchronize()
    print(f"7.5 MB H2D || 7.5 MB D2H: {a.elapsed_time(b) / 20 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
