"""GPU parity of the optimisation-ladder rungs (reference bench.py:35-41,
encoder.py:367-408): the padded baseline and the rm_padding rung against the
reference's frozen outputs, every rung against the fp32 oracle, and the padded
MHA kernel against the oracle's mha_padded."""

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


def _stress(bt, cfg, seed):
    ocfg = orc.OracleConfig(cfg.layers, cfg.head_num, 64, cfg.max_seq_len, cfg.batch_size)
    return bt.EncoderWeights(layers=[bt.encoder._layer_from_arrays(d) for d in orc.stress_weights(ocfg, seed)],
                             shared=False)


@pytest.mark.parametrize("tag,flags", [("tiny_padded", dict()), ("tiny_rmpad", dict(fuse_layernorm=True,
                                                                                   fuse_bias_gelu=True,
                                                                                   zero_padding=True))])
def test_ladder_golden(bt, golden, tag, flags):
    g = golden("encoder")
    cfg = bt.ModelConfig(layers=1, head_num=2, head_size=64, max_seq_len=40, batch_size=4, flags=bt.OptFlags(**flags))
    lens = g[f"{tag}_lengths"].tolist()
    x = orc.gen_input(lens, 40, 128, 4)
    y = bt.forward(_stress(bt, cfg, 4), bt.SeqLengths.of(lens, 40), bt.Tensor(x), cfg).array
    want = g[f"{tag}_out"]
    valid = orc.build_mask(lens, 40).reshape(-1).astype(bool)
    assert_close_bf16(y[valid], want[valid], max_abs_max=0.1 * rms(want[valid]), what=tag)
    if flags.get("zero_padding"):
        assert not y[~valid].any()
    else:  # the padded baseline computes padded rows too (reference semantics)
        assert_close_bf16(y[~valid], want[~valid], max_abs_max=0.1 * rms(want[~valid]), what=tag + " padded rows")


@pytest.mark.parametrize("name", ["baseline", "layernorm_fusion", "bias_gelu_fusion", "rm_padding", "fused_mha"])
def test_every_rung_matches_oracle(bt, name):
    from paper_2210_03052_b200.ladder import ladder_flags

    cfg = bt.preset_config("bert_base", 6, 160, ladder_flags(name), layers=2)
    lens = orc.gen_lengths(6, 160, "fixed", seed=1, alpha=0.6)
    x = orc.gen_input(lens, 160, 768, 1)
    w = _stress(bt, cfg, 2)
    y = bt.forward(w, bt.SeqLengths.of(lens, 160), bt.Tensor(x), cfg).array
    ocfg = orc.OracleConfig(2, 12, 64, 160, 6)
    want = orc.forward(orc.stress_weights(ocfg, 2), lens, x, ocfg)
    valid = orc.build_mask(lens, 160).reshape(-1).astype(bool)
    assert_close_bf16(y[valid], want[valid], max_abs_max=0.1 * rms(want[valid]), what=name)


def test_mha_padded_kernel(bt):
    import torch

    from paper_2210_03052_b200.ladder import mha_padded_device

    for mx, lens in ((200, [200, 1, 77, 129]), (600, [600, 3, 250])):
        plan = bt.plan_for_lengths(bt.SeqLengths.of(lens, mx))
        H = 2
        qkv = (torch.randn(len(lens) * mx, 3 * H * 64, device="cuda")).to(torch.bfloat16)
        out = mha_padded_device(qkv, plan, H, 64).float().cpu().numpy()
        a = qkv.float().cpu().numpy()
        z = np.zeros(H * 64, np.float32)
        want = orc.mha_padded(a[:, :128], a[:, 128:256], a[:, 256:], z, z, z, lens, mx, H, 64)
        assert_close_bf16(out, want, what=f"padded mha mx={mx}")
        valid = orc.build_mask(lens, mx).reshape(-1).astype(bool)
        assert not out[~valid].any()


def test_run_ladder_smoke(bt):
    from paper_2210_03052_b200.bench_ladder import BenchSpec, rows_to_csv, run_ladder

    res = run_ladder(BenchSpec(batch_size=4, max_seq_lens=(96,), alphas=(0.6,), mode="fixed", repeats=2, layers=2,
                               check=True))
    assert res.passed, res.diagnostics
    assert [r.variant for r in res.rows] == ["baseline", "layernorm_fusion", "bias_gelu_fusion", "rm_padding",
                                             "fused_mha"]
    assert rows_to_csv(res.rows).startswith("preset,variant,batch")
