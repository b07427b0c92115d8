"""Where the forward prologue's time goes (C2 by default): the one-launch
prologue against its pieces -- the single-CTA plan (bt_plan_forward) and the
pack alone (bt_pack_starts) -- each launched alone after an L2 flush by a READ
(as between bench steps) and after one by a WRITE (dirty L2), and 30 back to
back (L2-warm, launch overhead hidden behind a sleep).

    python scripts/prologue_probe.py [--config c2]
"""

import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    a = ap.parse_args()
    import torch

    import bench
    from paper_2210_03052_b200 import _lib, harness

    desc, heads, layers, bs, mx, _ = bench.WORKLOADS[a.config]
    k = heads * 64
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    T = seqs.total
    x = torch.from_numpy(harness.gen_input(seqs, k, 0)).cuda()
    lengths = torch.tensor(seqs.lengths, dtype=torch.int32, device="cuda")
    starts = torch.empty(bs + 1, dtype=torch.int32, device="cuda")
    sched = torch.empty(_lib.load().bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
    xp = torch.empty((T, k), dtype=torch.bfloat16, device="cuda")
    upad = torch.empty((bs * mx, k), dtype=torch.float32, device="cuda")
    row_map = torch.empty(T, dtype=torch.int32, device="cuda")
    S = _lib.stream_ptr
    ops = {
        "prologue": lambda: _lib.call("bt_forward_prologue", lengths.data_ptr(), bs, mx, k, x.data_ptr(), None,
                                      xp.data_ptr(), starts.data_ptr(), sched.data_ptr(), upad.data_ptr(),
                                      row_map.data_ptr(), T, S()),
        "plan_forward": lambda: _lib.call("bt_plan_forward", lengths.data_ptr(), bs, mx, starts.data_ptr(),
                                          sched.data_ptr(), S()),
        "pack_starts": lambda: _lib.call("bt_pack_starts", x.data_ptr(), starts.data_ptr(), bs, mx, k, xp.data_ptr(),
                                         S()),
        "empty_kernel": lambda: torch.cuda._sleep(0),
    }
    big = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    sink = torch.empty((), dtype=torch.float32, device="cuda")
    s = torch.cuda.current_stream()
    print(f"{a.config}: bs={bs} mx={mx} k={k} T={T}")
    for name, fn in ops.items():
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        out = {}
        for mode in ("read_flush", "write_flush"):
            reps = 20
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
            for e0, e1 in evs:
                if mode == "read_flush":
                    torch.sum(big, dim=0, out=sink)
                else:
                    big.fill_(1.0)
                e0.record(s)
                fn()
                e1.record(s)
            torch.cuda.synchronize()
            out[mode] = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in evs)[reps // 2]
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(int(2e7))
        e0.record(s)
        for _ in range(30):
            fn()
        e1.record(s)
        torch.cuda.synchronize()
        out["warm_b2b"] = e0.elapsed_time(e1) * 1e3 / 30
        print(f"  {name:14s} " + "  ".join(f"{m}={v:6.2f} us" for m, v in out.items()))


if __name__ == "__main__":
    main()
