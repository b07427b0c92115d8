"""Fused-MHA launch timing at C2 / C3 / C5 through bt_mha_varlen_sched (the
forward's schedule), back-to-back launches timed with CUDA events.
BT_LIB_PATH selects a library variant (A/B).

    python scripts/mha_time.py [c2 c3 c5 | bs:mx:heads ...]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.packing import plan_for_lengths

    _lib.require_device()
    for cfg in sys.argv[1:] or ["c2", "c3", "c5"]:
        known = {"c2": (16, 256, 12), "c3": (16, 512, 16), "c5": (2048, 512, 16)}
        bs, mx, H = known[cfg] if cfg in known else tuple(int(v) for v in cfg.split(":"))  # or "bs:mx:heads"
        seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
        plan = plan_for_lengths(seqs)
        T = plan.valid_word_cnt
        qkv = torch.randn(T, 3 * H * 64, device="cuda").to(torch.bfloat16)
        out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)
        sched = torch.zeros(_lib.load().bt_plan_sched_bytes(bs, mx) // 4 + 1, dtype=torch.int32, device="cuda")
        _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())

        def go():
            _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx,
                      H, 64, 384, out.data_ptr(), T, _lib.stream_ptr())

        n = 10 if cfg == "c5" else 200
        for _ in range(3 if cfg == "c5" else 50):
            go()
        torch.cuda.synchronize()
        res = []
        for _ in range(3):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            for _ in range(n):
                go()
            b.record()
            torch.cuda.synchronize()
            res.append(a.elapsed_time(b) * 1e3 / n)
        flops = 4.0 * sum(l * l for l in seqs.lengths) * 64 * H
        best = min(res)
        print(f"{cfg}: mha {best:.2f} us/launch (runs {' '.join(f'{r:.2f}' for r in res)}), "
              f"{flops / best / 1e6:.1f} TFLOP/s useful")


if __name__ == "__main__":
    main()
