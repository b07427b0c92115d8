"""GPU parity: mask -> plan -> pack/unpack kernels, bit-exact against the
oracle (which is pinned to the reference's golden vectors)."""

import numpy as np
import pytest

from oracle import packbert_np as orc

pytestmark = pytest.mark.gpu

CASES = ["fig4", "ones", "dense", "single", "r1", "r2", "r3"]


@pytest.fixture(scope="module")
def bt():
    import paper_2210_03052_b200 as bt

    bt._lib.require_device()
    return bt


@pytest.mark.parametrize("tag", CASES)
def test_plan_from_mask_bit_exact(bt, golden, tag):
    g = golden("packing")
    lens, mx = g[f"{tag}_lengths"], int(g[f"{tag}_mx"])
    plan = bt.compute_plan(orc.build_mask(lens, mx))
    np.testing.assert_array_equal(plan.offsets, g[f"{tag}_offsets"])
    np.testing.assert_array_equal(plan.seq_starts, g[f"{tag}_seq_starts"])
    assert plan.offsets.dtype == np.int64 and not plan.offsets.flags.writeable


@pytest.mark.parametrize("tag", CASES)
def test_plan_from_lengths_bit_exact(bt, golden, tag):
    g = golden("packing")
    lens, mx = g[f"{tag}_lengths"], int(g[f"{tag}_mx"])
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
    np.testing.assert_array_equal(plan.offsets, g[f"{tag}_offsets"])
    np.testing.assert_array_equal(plan.seq_starts, g[f"{tag}_seq_starts"])


def test_plan_c5_scale(bt, golden):
    """2048 sequences x 512 (C5): multi-chunk scan, 629,146 offsets."""
    lens = golden("generators")["c5_lengths"]
    offs, starts, _ = orc.compute_plan(orc.build_mask(lens, 512))
    plan = bt.compute_plan(orc.build_mask(lens, 512))
    assert plan.valid_word_cnt == len(offs) == 629146
    np.testing.assert_array_equal(plan.offsets, offs)
    np.testing.assert_array_equal(plan.seq_starts, starts)
    plan2 = bt.plan_for_lengths(bt.SeqLengths.of(lens, 512))
    np.testing.assert_array_equal(plan2.offsets, offs)


def test_plan_device_mask_validation(bt):
    import torch

    bad = torch.tensor([[1, 0, 1]], dtype=torch.uint8, device="cuda")
    with pytest.raises(bt.ShapeError, match="prefix"):
        bt.compute_plan(bad)
    with pytest.raises(bt.ShapeError, match="0 or 1"):
        bt.compute_plan(torch.tensor([[2, 0]], dtype=torch.uint8, device="cuda"))
    with pytest.raises(bt.ShapeError):
        bt.compute_plan(torch.tensor([[1, 1], [0, 0]], dtype=torch.uint8, device="cuda"))
    ok = bt.compute_plan(torch.tensor([[1, 1, 0], [1, 0, 0]], dtype=torch.uint8, device="cuda"))
    assert ok.offsets.tolist() == [0, 1, 3]
    with pytest.raises(bt.ShapeError):
        bt.compute_plan(np.array([[1, 0, 1]], np.uint8))


def test_pack_unpack_fp32_bit_exact(bt, golden):
    g = golden("packing")
    lens = g["pk_lengths"]
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, 40))
    packed = bt.pack(bt.Tensor(g["pk_padded"]), plan)
    np.testing.assert_array_equal(packed.tokens.array, g["pk_packed"])
    up = bt.unpack(packed, 40)
    np.testing.assert_array_equal(up.array, g["pk_unpacked"])
    with pytest.raises(bt.ShapeError):
        bt.unpack(packed, 41)
    with pytest.raises(bt.ShapeError):
        bt.pack(bt.Tensor(g["pk_padded"][:-1]), plan)


def test_unpack_fig4_zero_rows(bt):
    plan = bt.plan_for_lengths(bt.SeqLengths.of([2, 4, 5], 5))
    tokens = np.repeat(np.arange(11, dtype=np.float32)[:, None] + 1, 3, axis=1)
    up = bt.unpack(bt.PackedBatch(bt.Tensor(tokens), plan), 5).array
    assert [i for i in range(15) if not up[i].any()] == [2, 3, 4, 9]


def test_pack_bf16_and_round_trip_large(bt):
    """fp32 -> bf16 pack equals round-to-nearest of the fp32 gather; unpack
    restores every valid row and writes exact zeros elsewhere (C2 size)."""
    import torch

    lens = orc.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, 256))
    x = torch.randn(16 * 256, 768, device="cuda")
    from paper_2210_03052_b200.packing import pack_device, unpack_device

    pk = pack_device(x, plan, out_dtype=torch.bfloat16)
    idx = torch.from_numpy(plan.offsets).cuda()
    assert torch.equal(pk, x[idx].to(torch.bfloat16))
    up = unpack_device(pk, plan)
    ref = torch.zeros_like(x)
    ref[idx] = pk.float()
    assert torch.equal(up, ref)
    pk32 = pack_device(x, plan)
    assert torch.equal(unpack_device(pk32, plan)[idx], x[idx])


@pytest.mark.parametrize("bs,mx", [(16, 256), (1, 1), (300, 64), (2048, 512), (7, 1000)])
def test_forward_plan_and_pack_starts(bt, bs, mx):
    """The forward's one-launch plan (bt_plan_forward) gives plan_for_lengths'
    seq_starts bit for bit and the same MHA schedule as bt_plan_sched; the
    seq_starts-addressed pack (bt_pack_starts) equals the offsets pack."""
    import torch

    from paper_2210_03052_b200 import _lib
    from paper_2210_03052_b200.packing import pack_device

    lens = orc.gen_lengths(bs, mx, "fixed", seed=bs, alpha=0.6)
    seqs = bt.SeqLengths.of(lens, mx)
    plan = bt.plan_for_lengths(seqs)
    L = _lib.load()
    nb = L.bt_plan_sched_bytes(bs, mx) // 4
    sched_ref = torch.zeros(nb, dtype=torch.int32, device="cuda")
    sched = torch.full((nb,), -7, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_sched", plan.seq_starts_dev.data_ptr(), bs, mx, sched_ref.data_ptr(), _lib.stream_ptr())
    lengths_dev = torch.tensor(list(lens), dtype=torch.int32, device="cuda")
    starts = torch.full((bs + 1,), -1, dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_forward", lengths_dev.data_ptr(), bs, mx, starts.data_ptr(), sched.data_ptr(),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    assert np.array_equal(starts.cpu().numpy(), plan.seq_starts)
    # sequence order within a key-block bucket is unspecified: compare as multisets
    pairs = lambda t: sorted(map(tuple, t[:2 * bs].view(-1, 2).cpu().numpy().tolist()))  # noqa: E731
    assert pairs(sched) == pairs(sched_ref)
    off = (2 * bs * 4 + 15) // 16 * 4
    assert sched[off].item() == sched_ref[off].item()  # unit count
    k = 64
    x = torch.randn(bs * mx, k, device="cuda")
    out = torch.empty(plan.valid_word_cnt, k, dtype=torch.bfloat16, device="cuda")
    _lib.call("bt_pack_starts", x.data_ptr(), plan.seq_starts_dev.data_ptr(), bs, mx, k, out.data_ptr(),
              _lib.stream_ptr())
    torch.cuda.synchronize()
    assert torch.equal(out, pack_device(x, plan, out_dtype=torch.bfloat16))


def _segs_serial(lens):
    """The MHA segment list (plan_pack.cu plan_sched_body) as the serial greedy:
    long sequences' 128-row query tiles in order, then per run of adjacent
    sequences of <= 128 rows, groups closed when the next would pass 128 rows."""
    ss = np.concatenate([[0], np.cumsum(lens)]).astype(int)
    bs, out = len(lens), []
    for i in range(bs):
        st, en = ss[i], ss[i + 1]
        if en - st > 128:
            for q in range(st, en, 128):
                out.append((st, en, q, min(en, q + 128), i, i, 0, 0))
    g0 = -1
    for i in range(bs + 1):
        short = i < bs and ss[i + 1] - ss[i] <= 128
        if g0 >= 0 and (not short or ss[i + 1] - ss[g0] > 128):
            out.append((ss[g0], ss[i], ss[g0], ss[i], g0, i - 1, 0, 0))
            g0 = -1
        if short and g0 < 0:
            g0 = i
    return out


@pytest.mark.parametrize("case", ["mixed16", "all_short", "all_long", "edges", "bs256", "one", "mx64"])
def test_mha_segment_list(bt, case):
    """The parallel segment builder writes the serial greedy's list exactly,
    through all three launches that plan (bt_plan_sched, bt_plan_forward,
    bt_forward_prologue)."""
    import torch

    from paper_2210_03052_b200 import _lib

    rng = np.random.default_rng(len(case))
    lens, mx = {
        "mixed16": (orc.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6), 256),
        "all_short": (rng.integers(1, 129, 40), 128),
        "all_long": (rng.integers(129, 257, 12), 256),
        "edges": (np.array([128, 1, 127, 129, 64, 64, 1, 128, 256, 65, 63, 1, 1, 200, 128]), 256),
        "bs256": (rng.integers(1, 257, 256), 256),
        "one": (np.array([77]), 128),
        "mx64": (rng.integers(1, 65, 64), 64),
    }[case]
    lens = [int(v) for v in lens]
    bs, k = len(lens), 64
    want = _segs_serial(lens)
    L = _lib.load()
    nb = L.bt_plan_sched_bytes(bs, mx) // 4
    nbk = (mx + 127) // 128
    units_off = (bs * 8 + 15) // 16 * 16
    segs_off = (units_off + 16 + (bs * nbk * 8 + 15) // 16 * 16) // 4
    lengths_dev = torch.tensor(lens, dtype=torch.int32, device="cuda")
    starts = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int32, device="cuda")
    T = int(sum(lens))
    x = torch.randn(bs * mx, k, device="cuda")
    xp = torch.empty(T, k, dtype=torch.bfloat16, device="cuda")
    upad = torch.empty(bs * mx, k, device="cuda")
    row_map = torch.empty(T, dtype=torch.int32, device="cuda")
    st2 = torch.empty_like(starts)
    runs = {
        "plan_sched": lambda sc: _lib.call("bt_plan_sched", starts.data_ptr(), bs, mx, sc.data_ptr(),
                                           _lib.stream_ptr()),
        "plan_forward": lambda sc: _lib.call("bt_plan_forward", lengths_dev.data_ptr(), bs, mx, st2.data_ptr(),
                                             sc.data_ptr(), _lib.stream_ptr()),
        "prologue": lambda sc: _lib.call("bt_forward_prologue", lengths_dev.data_ptr(), bs, mx, k, x.data_ptr(), None,
                                         xp.data_ptr(), st2.data_ptr(), sc.data_ptr(), upad.data_ptr(),
                                         row_map.data_ptr(), T, _lib.stream_ptr()),
    }
    for name, run in runs.items():
        sched = torch.full((nb,), -7, dtype=torch.int32, device="cuda")
        run(sched)
        torch.cuda.synchronize()
        h = sched.cpu().numpy()
        n = int(h[segs_off])
        got = [tuple(int(v) for v in h[segs_off + 4 + 8 * i: segs_off + 12 + 8 * i]) for i in range(n)]
        assert n == len(want), (name, n, len(want))
        # the second int4's last two words are padding (not written)
        assert [g[:6] for g in got] == [w[:6] for w in want], name
