"""Forward-vs-oracle parity at the north-star geometries the other tests do
not reach (VERDICT r1 "what's missing" 2 / "next" 1):

* C3 geometry: BERT-large width (16 heads, k = 1024), batch 16, max_seq_len
  512 (> cutoff 384: the long-path MHA, reference attention.py:240-296),
  lengths gen_lengths(fixed, alpha 0.6, seed 0) -- 4 of the 24 layers, under
  the reference init and the stress init, through BOTH public entry points:
  ``forward(host Tensor)`` (cached CUDA graph of the packed forward, DMA of
  the valid rows) and ``forward(CUDA tensor)`` (``bt_encoder_forward``: the
  device plan + pack + layers + unpack that bench.py times).  The two must
  agree bit for bit, and each must match the fp32 oracle.
* C5 many-wave policy on a 64-sequence slice of the C5 batch: tile-list MHA
  (claim queue), several query tiles per CTA, multi-wave GEMMs -- vs the
  oracle, and bitwise equal to the default policy.
* PKBW weights: save_weights -> load_weights -> forward vs the oracle on the
  same file's weights (reference encoder.py:183-268 -> 411-437).

Tolerance (BASELINE.json north star): cosine >= 0.9999
and relFro <= 1.5e-2 always; max-abs <= 2e-2 under the reference init and
<= 0.1 * RMS(reference output) under the stress init."""

import numpy as np
import pytest

from oracle import packbert_np as orc
from tests._metrics import assert_close_bf16, rms

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bt():
    import paper_2210_03052_b200 as bt

    bt._lib.require_device()
    return bt


def _weights(bt, ocfg, seed, kind):
    wo = orc.init_weights(ocfg, seed) if kind == "init" else orc.stress_weights(ocfg, seed)
    return wo, bt.EncoderWeights(layers=[bt.encoder._layer_from_arrays(d) for d in wo],
                                 shared=ocfg.share_layer_weights)


def _check(bt, got, want, lens, mx, kind, what):
    valid = orc.build_mask(lens, mx).reshape(-1).astype(bool)
    g = np.asarray(got)
    if kind == "init":
        assert_close_bf16(g[valid], want[valid], max_abs_max=2e-2, what=what)
    else:
        assert_close_bf16(g[valid], want[valid], max_abs_max=0.1 * rms(want[valid]), what=what)
    assert not g[~valid].any(), f"{what}: padded rows must be exactly zero"


@pytest.mark.parametrize("kind", ["init", "stress"])
def test_forward_c3_geometry_vs_oracle(bt, kind):
    import torch

    bs, mx, heads, layers = 16, 512, 16, 4
    lens = orc.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
    x = orc.gen_input(lens, mx, heads * 64, 0)
    ocfg = orc.OracleConfig(layers, heads, 64, mx, bs)
    wo, w = _weights(bt, ocfg, 0, kind)
    want = orc.forward(wo, lens, x, ocfg)
    cfg = bt.ModelConfig(layers=layers, head_num=heads, head_size=64, max_seq_len=mx, batch_size=bs,
                         flags=bt.OptFlags.all_on())
    seqs = bt.SeqLengths.of(lens, mx)
    y_host = bt.forward(w, seqs, bt.Tensor(x), cfg).array
    y_dev = bt.forward(w, seqs, torch.from_numpy(x).cuda(), cfg).cpu().numpy()
    _check(bt, y_host, want, lens, mx, kind, f"C3 {kind} host path")
    _check(bt, y_dev, want, lens, mx, kind, f"C3 {kind} device path (bt_encoder_forward)")
    assert np.array_equal(y_host, y_dev), "host-DMA graph path and bt_encoder_forward must agree bitwise"


def test_forward_c5_slice_many_wave_vs_oracle(bt):
    """The many-wave policies forced on a 64-sequence slice of the C5 batch."""
    import torch

    from paper_2210_03052_b200 import _lib

    mx, heads, layers = 512, 16, 2
    lens = orc.gen_lengths(2048, mx, "fixed", seed=0, alpha=0.6)[:64]
    bs = len(lens)
    x = orc.gen_input(lens, mx, heads * 64, 1)
    ocfg = orc.OracleConfig(layers, heads, 64, mx, bs)
    wo, _ = _weights(bt, ocfg, 1, "stress")
    want = orc.forward(wo, lens, x, ocfg)
    cfg = bt.ModelConfig(layers=layers, head_num=heads, head_size=64, max_seq_len=mx, batch_size=bs,
                         flags=bt.OptFlags.all_on())
    seqs = bt.SeqLengths.of(lens, mx)
    xd = torch.from_numpy(x).cuda()
    outs = {}
    try:
        # the default: the four-CTA MHA (mha64_sm100.cu), one tile per CTA
        _, w = _weights(bt, ocfg, 1, "stress")
        y64 = bt.forward(w, seqs, xd, cfg).cpu().numpy()
        # the two-CTA kernels' many-wave modes (mha_sm100.cu), pinned bitwise
        # against each other
        _lib.call("bt_debug_mha64", 0)
        for name, (list_mode, grid, qg) in {"default": (-1, 0, 0), "tile_list": (2, 0, 0),
                                            "tile_list_small_grid": (2, 37, 0), "qg4": (0, 0, 4)}.items():
            _lib.call("bt_debug_mha_list", list_mode, grid)
            _lib.call("bt_debug_mha_qg", qg)
            _, w = _weights(bt, ocfg, 1, "stress")  # fresh engine per policy
            outs[name] = bt.forward(w, seqs, xd, cfg).cpu().numpy()
    finally:
        _lib.call("bt_debug_mha_list", -1, 0)
        _lib.call("bt_debug_mha_qg", 0)
        _lib.call("bt_debug_mha64", -1)
    _check(bt, y64, want, lens, mx, "stress", "C5 slice, four-CTA MHA")
    _check(bt, outs["tile_list"], want, lens, mx, "stress", "C5 slice, tile list")
    for name, y in outs.items():
        assert np.array_equal(y, outs["default"]), f"{name} differs from the two-CTA default policy"


def test_pkbw_weights_forward_vs_oracle(bt, tmp_path):
    """save_weights -> load_weights -> device upload -> forward, vs the oracle
    run on the arrays read back from the same file."""
    import torch

    cfg = bt.preset_config("bert_base", 5, 300, bt.OptFlags.all_on(), layers=2)
    w0 = bt.init_weights(cfg, seed=7)
    path = tmp_path / "w.pkbw"
    bt.save_weights(path, w0, cfg)
    w = bt.load_weights(path, cfg)
    lens = [300, 17, 128, 1, 256]
    x = orc.gen_input(lens, 300, 768, 7)
    ocfg = orc.OracleConfig(2, 12, 64, 300, 5)
    wo = [bt.encoder._layer_arrays(lw) for lw in w.layers]
    want = orc.forward(wo, lens, x, ocfg)
    y = bt.forward(w, bt.SeqLengths.of(lens, 300), torch.from_numpy(x).cuda(), cfg).cpu().numpy()
    _check(bt, y, want, lens, 300, "init", "PKBW -> device")
    # and the loaded weights are the saved ones, bit for bit
    y0 = bt.forward(w0, bt.SeqLengths.of(lens, 300), torch.from_numpy(x).cuda(), cfg).cpu().numpy()
    assert np.array_equal(y, y0)
