"""MHA launch timing, tile-list mode vs one tile per CTA: isolated launches
(synchronised, events around one launch) and back-to-back launches.

    python scripts/mha_list_timing.py c2|c3
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.packing import plan_for_lengths

    _lib.require_device()
    bs, mx, H = {"c2": (16, 256, 12), "c3": (16, 512, 16), "c5": (2048, 512, 16)}[sys.argv[1]]
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    plan = plan_for_lengths(seqs)
    T = plan.valid_word_cnt
    qkv = torch.randn(T, 3 * H * 64, device="cuda").to(torch.bfloat16)
    out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)
    sched = torch.zeros(_lib.load().bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
    s = torch.cuda.current_stream()

    def go():
        _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx, H,
                  64, 384, out.data_ptr(), T, _lib.stream_ptr())

    for mode in (0, 1, 0, 1):
        _lib.call("bt_debug_mha_list", mode, 0)
        for _ in range(300):
            go()
        torch.cuda.synchronize()
        iso = []
        for _ in range(50):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record(s)
            go()
            b.record(s)
            torch.cuda.synchronize()
            iso.append(a.elapsed_time(b) * 1e3)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(100):
            go()
        b.record(s)
        torch.cuda.synchronize()
        print(f"{sys.argv[1]} list={mode}: isolated median {np.median(iso):.2f} us (min {min(iso):.2f}); "
              f"back-to-back {a.elapsed_time(b) * 10:.2f} us/launch")
    _lib.call("bt_debug_mha_list", -1, 0)


if __name__ == "__main__":
    main()
