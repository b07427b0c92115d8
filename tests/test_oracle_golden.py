"""Pin the CPU oracle (oracle/packbert_np.py) to the reference's own outputs
frozen in tests/golden/*.npz by tests/golden/make_golden.py."""

import math

import numpy as np
import pytest

from oracle import packbert_np as orc


def _rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    d = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (d if d else 1.0)


@pytest.mark.parametrize("tag", ["fig4", "ones", "dense", "single", "r1", "r2", "r3"])
def test_plan_bit_exact(golden, tag):
    g = golden("packing")
    lens, mx = g[f"{tag}_lengths"], int(g[f"{tag}_mx"])
    offs, starts, got_lens = orc.compute_plan(orc.build_mask(lens, mx))
    assert offs.dtype == np.int64 and starts.dtype == np.int64
    np.testing.assert_array_equal(offs, g[f"{tag}_offsets"])
    np.testing.assert_array_equal(starts, g[f"{tag}_seq_starts"])
    np.testing.assert_array_equal(got_lens, lens)


def test_plan_kats():
    # SPEC.md:120,130,132 (Fig. 4 and the [1,1]/4 case)
    offs, starts, _ = orc.compute_plan(orc.build_mask([2, 4, 5], 5))
    assert offs.tolist() == [0, 1, 5, 6, 7, 8, 10, 11, 12, 13, 14]
    assert starts.tolist() == [0, 2, 6, 11]
    offs, _, _ = orc.compute_plan(orc.build_mask([1, 1], 4))
    assert offs.tolist() == [0, 4]


def test_plan_rejects_bad_masks():
    with pytest.raises(ValueError):
        orc.compute_plan(np.array([[1, 0, 1]], np.uint8))
    with pytest.raises(ValueError):
        orc.compute_plan(np.array([[2, 0, 0]], np.uint8))
    with pytest.raises(ValueError):
        orc.compute_plan(np.zeros((2, 2, 2), np.uint8))


def test_pack_unpack_bit_exact(golden):
    g = golden("packing")
    lens = g["pk_lengths"]
    offs, _, _ = orc.compute_plan(orc.build_mask(lens, 40))
    packed = orc.pack(g["pk_padded"], offs)
    np.testing.assert_array_equal(packed, g["pk_packed"])
    np.testing.assert_array_equal(orc.unpack(packed, offs, len(lens) * 40), g["pk_unpacked"])
    # Fig. 4 padded rows {2,3,4,9} are exactly zero
    u = g["fig4_unpacked"]
    zero_rows = [i for i in range(15) if not u[i].any()]
    assert zero_rows == [2, 3, 4, 9]


def test_generators(golden):
    g = golden("generators")
    for tag, (bs, mx) in {"c1": (16, 128), "c2": (16, 256), "c3": (16, 512), "c5": (2048, 512)}.items():
        lens = orc.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
        assert lens == g[f"{tag}_lengths"].tolist(), tag
        assert sum(lens) == round(0.6 * bs * mx)
    assert orc.gen_lengths(50, 77, "uniform", seed=4) == g["uniform_lengths"].tolist()
    lens = g["input_lengths"].tolist()
    np.testing.assert_array_equal(orc.gen_input(lens, 16, 32, seed=2), g["input_x"])
    cfg = orc.OracleConfig(layers=2, head_num=2, head_size=8, max_seq_len=16, batch_size=4)
    for li, layer in enumerate(orc.init_weights(cfg, seed=3)):
        for name, arr in layer.items():
            np.testing.assert_array_equal(arr, g[f"w{li}_{name}"])
    c2 = orc.exact_flops(g["c2_lengths"].tolist(), 768)
    for key, val in c2.items():
        assert val == int(g[f"flops_c2_{key}"])
    # SPEC.md:515 Table II KAT is for the analytic model; the exact C2 model
    # above must equal 24 T k^2 + 4 sum(len^2) k per layer.
    T = sum(g["c2_lengths"].tolist())
    assert sum(c2.values()) == 24 * T * 768 ** 2 + 4 * sum(n * n for n in g["c2_lengths"].tolist()) * 768


def test_fusion(golden):
    g = golden("fusion")
    np.testing.assert_array_equal(orc.gelu(g["gelu_in"]), g["gelu_out"])
    y = orc.add_bias_residual_layernorm(g["ln_x"], g["ln_r"], g["ln_b"], g["ln_g"], g["ln_beta"])
    np.testing.assert_array_equal(y, g["ln_y"])
    np.testing.assert_allclose(g["ln_kat"], [[-1.224745, 0.0, 1.224745]], atol=1e-6)
    assert abs(float(orc.gelu(np.float32(1.0))) - 0.841192) < 1e-6


@pytest.mark.parametrize("tag", ["short", "long", "cut384", "cut385"])
def test_attention(golden, tag):
    g = golden("attention")
    lens = g[f"{tag}_lengths"].tolist()
    mx, heads = int(g[f"{tag}_mx"]), int(g[f"{tag}_heads"])
    _, starts, _ = orc.compute_plan(orc.build_mask(lens, mx))
    o = orc.dispatch_mha(g[f"{tag}_q"], g[f"{tag}_k"], g[f"{tag}_v"], g[f"{tag}_bias"], starts, mx, heads, 64)
    # same numpy ops in the same order -> bitwise on this host's BLAS
    assert _rel(o, g[f"{tag}_out"]) <= 1e-6


def test_dispatch_boundary():
    # 384 -> short path, 385 -> long path
    lens = [3, 2]
    q = np.random.default_rng(0).standard_normal((5, 64)).astype(np.float32)
    b = np.zeros(192, np.float32)
    _, st, _ = orc.compute_plan(orc.build_mask(lens, 384))
    a = orc.dispatch_mha(q, q, q, b, st, 384, 1, 64)
    c = orc.dispatch_mha(q, q, q, b, st, 385, 1, 64)
    assert _rel(a, c) < 1e-6


@pytest.mark.parametrize("tag,layers,heads,mx,bs,seed,flags,wkind", [
    ("tiny", 2, 2, 48, 6, 0, {}, "init"),
    ("tiny_long", 1, 2, 400, 3, 1, {}, "init"),
    ("tiny_stress", 2, 2, 96, 5, 2, {}, "stress"),
    ("tiny_stress_long", 1, 2, 450, 2, 3, {}, "stress"),
    ("tiny_padded", 1, 2, 40, 4, 4, dict(fuse_layernorm=False, fuse_bias_gelu=False, zero_padding=False,
                                          fused_mha=False), "stress"),
    ("tiny_rmpad", 1, 2, 40, 4, 4, dict(fused_mha=False), "stress"),
])
def test_encoder_forward(golden, tag, layers, heads, mx, bs, seed, flags, wkind):
    g = golden("encoder")
    cfg = orc.OracleConfig(layers, heads, 64, mx, bs)
    lens = orc.gen_lengths(bs, mx, "fixed", seed=seed, alpha=0.6)
    assert lens == g[f"{tag}_lengths"].tolist()
    x = orc.gen_input(lens, mx, cfg.hidden, seed)
    w = orc.init_weights(cfg, seed) if wkind == "init" else orc.stress_weights(cfg, seed)
    y = orc.forward(w, lens, x, cfg, **flags)
    assert _rel(y, g[f"{tag}_out"]) <= 1e-6
    if flags.get("zero_padding", True):
        pad = ~orc.build_mask(lens, mx).reshape(-1).astype(bool)
        assert not y[pad].any()


@pytest.mark.slow
def test_encoder_c1(golden):
    g = golden("encoder")
    cfg = orc.OracleConfig(1, 12, 64, 128, 16)
    lens = orc.gen_lengths(16, 128, "fixed", seed=0, alpha=0.6)
    y = orc.forward(orc.init_weights(cfg, 0), lens, orc.gen_input(lens, 128, 768, 0), cfg)
    assert _rel(y[g["c1_rows"]], g["c1_out_sub"]) <= 1e-6
    assert math.isclose(float(np.linalg.norm(y.astype(np.float64))), float(g["c1_out_norm"]), rel_tol=1e-6)
