"""One small launch of every MHA scheduling mode, the forward plan, the
seq_starts pack and the one-launch prologue, for compute-sanitizer runs:

    compute-sanitizer --tool memcheck python scripts/sanitize_mha.py
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch

    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200 import _lib

    _lib.require_device()
    L = _lib.load()
    # the third batch has enough query tiles x heads (> 16 x SMs) for the
    # four-CTA MHA's persistent mode
    for lens, mx, H in (([5, 300, 129, 1, 200, 128, 77], 512, 2), ([1, 2, 3, 127, 128, 129, 200, 256, 30, 40], 256, 2),
                        ([512, 511, 385, 200, 64, 1] * 7, 512, 16)):
        bs = len(lens)
        plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
        T = plan.valid_word_cnt
        qkv = torch.randn(T, 3 * H * 64, device="cuda").to(torch.bfloat16)
        out = torch.empty(T, H * 64, device="cuda", dtype=torch.bfloat16)
        sched = torch.zeros(L.bt_plan_sched_bytes(bs, mx) // 4, dtype=torch.int32, device="cuda")
        lengths = torch.tensor(lens, dtype=torch.int32, device="cuda")
        starts = torch.empty(bs + 1, dtype=torch.int32, device="cuda")
        _lib.call("bt_plan_forward", lengths.data_ptr(), bs, mx, starts.data_ptr(), sched.data_ptr(), _lib.stream_ptr())
        x = torch.randn(bs * mx, 64, device="cuda")
        pk = torch.empty(T, 64, device="cuda", dtype=torch.bfloat16)
        _lib.call("bt_pack_starts", x.data_ptr(), starts.data_ptr(), bs, mx, 64, pk.data_ptr(), _lib.stream_ptr())
        # the one-launch prologue (plan + segment list + pack + zero rows)
        upad = torch.empty(bs * mx, 64, device="cuda")
        row_map = torch.empty(T, dtype=torch.int32, device="cuda")
        sched2 = torch.zeros_like(sched)
        _lib.call("bt_forward_prologue", lengths.data_ptr(), bs, mx, 64, x.data_ptr(), None, pk.data_ptr(),
                  starts.data_ptr(), sched2.data_ptr(), upad.data_ptr(), row_map.data_ptr(), T, _lib.stream_ptr())
        for m64, seg, lst, grid in ((1, 0, 0, 0), (0, 0, 0, 0), (0, 2, 0, 0), (0, 0, 2, 0), (0, 0, 2, 3)):
            _lib.call("bt_debug_mha64", m64)  # the four-CTA kernel, then the two-CTA kernels' modes
            _lib.call("bt_debug_mha_seg", seg)
            _lib.call("bt_debug_mha_list", lst, grid)
            _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), starts.data_ptr(), sched.data_ptr(), bs, mx, H, 64, 384,
                      out.data_ptr(), T, _lib.stream_ptr())
            torch.cuda.synchronize()
        _lib.call("bt_debug_mha64", -1)
        _lib.call("bt_debug_mha_seg", -1)
        _lib.call("bt_debug_mha_list", -1, 0)
    print("sanitize run done")


if __name__ == "__main__":
    main()
