"""Run single MHA launches through BT_MHA64=1 (one case per process: argv =
mx H lens...), print OK / max diff against the default kernel."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2210_03052_b200 as bt
    from paper_2210_03052_b200.attention import mha_device
    mx, H = int(sys.argv[1]), int(sys.argv[2])
    lens = [int(x) for x in sys.argv[3:]]
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    g = torch.Generator(device="cuda").manual_seed(3)
    qkv = (torch.randn(plan.valid_word_cnt, 3 * H * 64, device="cuda", generator=g)).to(torch.bfloat16)
    out = mha_device(qkv, plan, H, 64)
    torch.cuda.synchronize()
    print("launched", flush=True)
    print(f"mx={mx} H={H} lens={lens}: finite={torch.isfinite(out.float()).all().item()}", flush=True)


if __name__ == "__main__":
    main()
