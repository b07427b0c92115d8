"""Per-CTA phase timeline of one four-CTA MHA launch (mha64_sm100.cu, grid
mode), globaltimer ns.

    python scripts/mha64_trace.py c2|c3|BS:MX:HEADS

Needs a trace build (the trace points are compiled out otherwise):
    python -c "from paper_2210_03052_b200 import build; build.build_variant('abv/trace.so', ['BT_TRACE_ON'])"
    BT_LIB_PATH=abv/trace.so python scripts/mha64_trace.py c2

Phases per 64-key block j (medians over the CTAs with >= 2 blocks):
  softmax   S(j) seen -> P(j) released (registers, exponentials, P store)
  mma_wake  P(j) released -> the MMA warp sees it (mbarrier round trip)
  mma_rt    P(j) released -> S(j+1) seen by the softmax (P V(j) + S(j+1) MMAs
            and their commit)
"""

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch

    from paper_2210_03052_b200 import _lib, harness
    from paper_2210_03052_b200.attention import mha_device
    from paper_2210_03052_b200.packing import plan_for_lengths

    _lib.require_device()
    spec = sys.argv[1]
    named = {"c2": (16, 256, 12), "c3": (16, 512, 16)}
    bs, mx, H = named[spec] if spec in named else tuple(int(v) for v in spec.split(":"))
    seqs = harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    plan = plan_for_lengths(seqs)
    qkv = torch.randn(plan.valid_word_cnt, 3 * H * 64, device="cuda").to(torch.bfloat16)
    _lib.call("bt_debug_mha64", 1)
    _lib.call("bt_debug_mha_seg", 0)
    for _ in range(2000):  # clocks up to their loaded level before the traced launch
        mha_device(qkv, plan, H, 64)
    nq = (mx + 127) // 128
    n = nq * H * bs
    buf = torch.zeros(n * 32, dtype=torch.int64, device="cuda")
    _lib.call("bt_debug_mha_trace", buf.data_ptr())
    mha_device(qkv, plan, H, 64)
    torch.cuda.synchronize()
    _lib.call("bt_debug_mha_trace", 0)
    _lib.call("bt_debug_mha64", -1)
    _lib.call("bt_debug_mha_seg", -1)
    t = buf.view(n, 32).cpu().numpy().astype(np.float64)
    used = t[:, 0] > 0
    t0 = t[used, 0].min()
    us = lambda x: (x - t0) / 1e3  # noqa: E731
    print(f"{spec}: bs {bs} mx {mx} heads {H}; CTAs with a tile {used.sum()} of {n}; "
          f"set-up done {us(t[used, 0]).min():.2f}..{us(t[used, 0]).max():.2f} us; "
          f"stored {us(t[used, 31]).min():.2f}..{us(t[used, 31]).max():.2f} us")
    lens = seqs.lengths
    ph = {"setup->Q": [], "Q->S0": [], "softmax": [], "mma_wake": [], "mma_rt": [], "lastP->O": [], "O->stored": []}
    for c in np.nonzero(used)[0]:
        row = t[c]
        b = c // (H * nq)
        nkb = (lens[b] + 63) // 64
        ph["setup->Q"].append(row[1] - row[0])
        ph["Q->S0"].append(row[2] - row[1])
        last = min(nkb, 7) - 1
        for j in range(min(nkb, 7)):
            ph["softmax"].append(row[3 + 2 * j] - row[2 + 2 * j])
            ph["mma_wake"].append(row[16 + j] - row[3 + 2 * j])
            if j + 1 < min(nkb, 7):
                ph["mma_rt"].append(row[2 + 2 * (j + 1)] - row[3 + 2 * j])
        if nkb <= 7:
            ph["lastP->O"].append(row[30] - row[3 + 2 * last])
        ph["O->stored"].append(row[31] - row[30])
    for k, v in ph.items():
        if v:
            v = np.array(v) / 1e3
            print(f"  {k:10s} median {np.median(v):6.3f} us  p90 {np.percentile(v, 90):6.3f}  n {len(v)}")
    longest = max(np.nonzero(used)[0], key=lambda c: t[c, 31] - t0)
    row = t[longest]
    b = longest // (H * nq)
    s = f"  last CTA to finish (len {lens[b]}): setup {us(row[0]):.2f} Q {us(row[1]):.2f} |"
    for j in range(7):
        if row[2 + 2 * j] == 0:
            break
        s += f" S{j} {us(row[2 + 2 * j]):.2f}-{us(row[3 + 2 * j]):.2f}"
    print(s + f" | O {us(row[30]):.2f} stored {us(row[31]):.2f}")


if __name__ == "__main__":
    main()
