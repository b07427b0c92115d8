"""The persistent fused varlen MHA the forward runs (csrc/mha2_sm100.cu):
parity with the fp32 oracle (reference attention.py:177-314) on edge
lengths, grouped short sequences, long sequences and a late max jump;
results independent of the grid (any number of CTAs claiming units from the
queue, which every launch leaves reset); a sequence's output independent of
its neighbours; and the launch-instrumented FLOP count."""

import numpy as np
import pytest

from oracle import packbert_np as orc
from tests._metrics import assert_close_bf16

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def env():
    import torch

    import paper_2210_03052_b200 as bt

    bt._lib.require_device()
    return bt, torch


def _rand_qkv(torch, T, hid, scale=1.0, seed=0):
    gen = torch.Generator(device="cuda").manual_seed(seed)
    return (torch.randn(T, 3 * hid, device="cuda", generator=gen) * scale).to(torch.bfloat16)


def _oracle(qkv, plan, heads, mx, cutoff=384):
    a = qkv.float().cpu().numpy()
    hid = heads * 64
    zero = np.zeros(3 * hid, np.float32)
    return orc.dispatch_mha(a[:, :hid], a[:, hid:2 * hid], a[:, 2 * hid:], zero, plan.seq_starts, mx, heads, 64,
                            cutoff)


def _mha2(bt, torch, qkv, plan, heads, mx):
    """The forward's MHA call: bt_plan_sched schedule + bt_mha_varlen_sched."""
    from paper_2210_03052_b200 import _lib

    bs, T = plan.batch_size, plan.valid_word_cnt
    sched = torch.full((_lib.load().bt_plan_sched_bytes(bs, mx) // 4,), -1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched.data_ptr(), _lib.stream_ptr())
    out = torch.full((T, heads * 64), float("nan"), device="cuda", dtype=torch.bfloat16)
    _lib.call("bt_mha_varlen_sched", qkv.data_ptr(), plan.seq_starts_dev.data_ptr(), sched.data_ptr(), bs, mx, heads,
              64, 384, out.data_ptr(), T, _lib.stream_ptr())
    torch.cuda.synchronize()
    return out


CASES = [
    ([1, 2, 3, 127, 128, 129, 200, 256], 256),  # tile edges, grouped short sequences
    ([384, 1, 383, 257, 77], 384),  # the cutoff, short path in the reference
    ([385, 5, 512, 129, 1, 640], 640),  # long path
    ([5] * 40, 8),  # many tiny sequences in groups
    ([1] * 250 + [64, 250], 256),  # groups of hundreds of 1-token sequences
    ([1000, 3, 700, 129], 1024),
    ([244, 190, 157, 96, 105, 36, 45, 30, 70, 234, 192, 256, 154, 181, 256, 212], 256),  # the C2 batch
    ([64] * 300, 64),  # > 256 sequences: no groups
]


@pytest.mark.parametrize("lens,mx", CASES)
def test_mha2_vs_oracle(env, lens, mx):
    bt, torch = env
    heads = 3
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=len(lens) + mx)
    out = _mha2(bt, torch, qkv, plan, heads, mx)
    assert torch.isfinite(out.float()).all()
    assert_close_bf16(out, _oracle(qkv, plan, heads, mx), what=f"mha2 {lens[:4]} mx={mx}")


def test_mha2_reference_max_moves(env):
    """A late jump of the row max (keys 128.. scaled 4x) forces the lazy
    reference max to move and O / the row sum to be rescaled."""
    bt, torch = env
    lens, mx, heads = [37, 200, 5, 512, 90, 1, 300], 512, 2
    hid = heads * 64
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, hid, seed=21)
    s = plan.seq_starts
    for b in range(len(lens)):
        lo, hi = s[b] + 128, s[b + 1]
        if hi > lo:
            qkv[lo:hi, hid:2 * hid] *= 4
    out = _mha2(bt, torch, qkv, plan, heads, mx)
    assert_close_bf16(out, _oracle(qkv, plan, heads, mx), what="mha2 rescale")


@pytest.mark.parametrize("lens,mx", [CASES[2], CASES[4], CASES[6], CASES[7]])
def test_mha2_grid_invariance(env, lens, mx):
    """One CTA walking every unit, a few CTAs, more CTAs than units, the
    default grid -- and repeated launches (the claim queue is reset by each
    launch) -- all give the same bits."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib

    heads = 2
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=7)
    ref = _mha2(bt, torch, qkv, plan, heads, mx)
    try:
        for grid in (1, 3, 37, 5000, 0):
            _lib.call("bt_debug_mha2_grid", grid)
            for _ in range(2):
                assert torch.equal(_mha2(bt, torch, qkv, plan, heads, mx), ref), f"grid {grid}"
    finally:
        _lib.call("bt_debug_mha2_grid", 0)


def test_mha2_isolation(env):
    """Perturbing every other sequence's q/k/v leaves a sequence's output
    bitwise unchanged (max_seq_len > 256: every sequence on its own tiles)."""
    bt, torch = env
    lens, mx, heads = [37, 300, 5, 512, 90, 1, 140], 512, 2
    hid = heads * 64
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, hid, seed=23)
    out = _mha2(bt, torch, qkv, plan, heads, mx)
    s = plan.seq_starts
    for keep in (0, 1, 5):
        pert = qkv.clone()
        for b in range(len(lens)):
            if b != keep:
                pert[s[b]:s[b + 1]] = (torch.randn_like(pert[s[b]:s[b + 1]].float()) * 3).to(torch.bfloat16)
        out2 = _mha2(bt, torch, pert, plan, heads, mx)
        assert torch.equal(out[s[keep]:s[keep + 1]], out2[s[keep]:s[keep + 1]]), keep


def test_mha2_matches_per_policy_kernels(env):
    """The persistent kernel and the one-tile-per-CTA kernels it replaced agree
    to bf16 rounding on a forward (C2 geometry, 2 layers)."""
    bt, torch = env
    from paper_2210_03052_b200 import _lib

    lens = orc.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on(), layers=2)
    x = torch.from_numpy(orc.gen_input(lens, 256, 768, 0)).cuda()
    seqs = bt.SeqLengths.of(lens, 256)
    y2 = bt.forward(bt.init_weights(cfg, 0), seqs, x, cfg)
    _lib.call("bt_debug_mha_v2", 0)
    try:
        y1 = bt.forward(bt.init_weights(cfg, 0), seqs, x, cfg)
    finally:
        _lib.call("bt_debug_mha_v2", -1)
    assert_close_bf16(y2, y1, what="mha2 vs per-policy kernels")


def test_mha2_flop_instrumentation(env):
    bt, torch = env
    from paper_2210_03052_b200.instrument import LaunchFlops

    lens, mx, heads = [1, 2, 3, 127, 128, 129, 200, 256], 256, 3
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    qkv = _rand_qkv(torch, plan.valid_word_cnt, heads * 64, seed=1)
    with LaunchFlops() as lf:
        _mha2(bt, torch, qkv, plan, heads, mx)
    assert lf.counts["mha"] == sum(4 * n * n * 64 for n in lens) * heads
