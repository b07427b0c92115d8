"""Host-side API parity with the reference (no GPU needed): containers,
init, config parsing, weight files, validation, error types."""

import numpy as np
import pytest

import paper_2210_03052_b200 as bt
from oracle import packbert_np as orc


def test_error_hierarchy():
    assert issubclass(bt.ShapeError, ValueError) and issubclass(bt.ShapeError, bt.PackbertError)
    assert issubclass(bt.ConfigError, ValueError)
    assert issubclass(bt.WeightFormatError, ValueError)


def test_seq_lengths_validation():
    s = bt.SeqLengths.of([2, 4, 5], 5)
    assert s.total == 11 and s.batch_size == 3 and abs(s.alpha - 11 / 15) < 1e-12
    with pytest.raises(bt.ShapeError):
        bt.SeqLengths.of([], 5)
    with pytest.raises(bt.ShapeError):
        bt.SeqLengths.of([0, 3], 5)
    with pytest.raises(bt.ShapeError):
        bt.SeqLengths.of([6], 5)
    with pytest.raises(bt.ShapeError):
        bt.SeqLengths.of([1], 0)


def test_build_mask_kat():
    m = bt.build_mask(bt.SeqLengths.of([2, 4, 5], 5))
    assert m.dtype == np.uint8
    assert m.tolist() == [[1, 1, 0, 0, 0], [1, 1, 1, 1, 0], [1, 1, 1, 1, 1]]


def test_model_config_validation():
    with pytest.raises(bt.ConfigError):
        bt.ModelConfig(layers=0, head_num=1, head_size=64, max_seq_len=8, batch_size=1)
    with pytest.raises(bt.ConfigError):
        bt.ModelConfig(layers=1, head_num=1, head_size=64, max_seq_len=8, batch_size=1,
                       flags=bt.OptFlags(fused_mha=True))
    c = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
    assert c.hidden_dim == 768 and c.layers == 12 and c.cutoff == 384 and c.split_seq_len == 32
    assert bt.preset_config("albert", 1, 8).share_layer_weights
    with pytest.raises(bt.ConfigError):
        bt.preset_config("gpt", 1, 8)


def test_init_weights_match_reference(golden):
    g = golden("generators")
    cfg = bt.ModelConfig(layers=2, head_num=2, head_size=8, max_seq_len=16, batch_size=4)
    w = bt.init_weights(cfg, seed=3)
    for li in range(2):
        lw = w.layer(li)
        np.testing.assert_array_equal(lw.qkv_weight, g[f"w{li}_qkv_weight"])
        np.testing.assert_array_equal(lw.ffn_w2, g[f"w{li}_ffn_w2"])
        np.testing.assert_array_equal(lw.ln1.beta, g[f"w{li}_ln1_beta"])
    shared = bt.init_weights(bt.preset_config("albert", 1, 8, layers=3), 0)
    assert len(shared.layers) == 1 and shared.layer(2) is shared.layer(0)


def test_pkbw_round_trip_and_validation(tmp_path):
    cfg = bt.ModelConfig(layers=2, head_num=2, head_size=8, max_seq_len=16, batch_size=4)
    w = bt.init_weights(cfg, seed=1)
    p = tmp_path / "w.pkbw"
    bt.save_weights(p, w, cfg)
    w2 = bt.load_weights(p, cfg)
    for a, b in zip(w.layers, w2.layers):
        np.testing.assert_array_equal(a.qkv_weight, b.qkv_weight)
        np.testing.assert_array_equal(a.ln0.gamma, b.ln0.gamma)
    raw = p.read_bytes()
    (tmp_path / "bad_magic").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(bt.WeightFormatError, match="bad magic"):
        bt.load_weights(tmp_path / "bad_magic", cfg)
    (tmp_path / "short").write_bytes(raw[:-4])
    with pytest.raises(bt.WeightFormatError, match="payload"):
        bt.load_weights(tmp_path / "short", cfg)
    with pytest.raises(bt.WeightFormatError, match="layers"):
        bt.load_weights(p, bt.ModelConfig(layers=3, head_num=2, head_size=8, max_seq_len=16, batch_size=4))
    (tmp_path / "tiny").write_bytes(b"PK")
    with pytest.raises(bt.WeightFormatError, match="too short"):
        bt.load_weights(tmp_path / "tiny", cfg)


def test_parse_config():
    cfg = bt.parse_config_text("""
        # BERT-base padding-free
        layers = 12
        head_num=12
        head_size=64
        max_seq_len=256
        batch_size=16
        fuse_layernorm=on
        fuse_bias_gelu=yes
        zero_padding=1
        fused_mha=true
    """)
    assert cfg.flags == bt.OptFlags.all_on() and cfg.hidden_dim == 768
    with pytest.raises(bt.ConfigError, match="unknown config key"):
        bt.parse_config_text("layers=1\nbogus=2")
    with pytest.raises(bt.ConfigError, match="missing required"):
        bt.parse_config_text("layers=1")
    with pytest.raises(bt.ConfigError, match="integer"):
        bt.parse_config_text("layers=x")
    with pytest.raises(bt.ConfigError, match="boolean"):
        bt.parse_config_text("layers=1\nhead_num=1\nhead_size=64\nmax_seq_len=4\nbatch_size=1\nfused_mha=maybe")


def test_forward_validates_before_compute():
    """Shape errors are raised on the host, before any device work (no GPU here)."""
    cfg = bt.preset_config("bert_base", 2, 8, bt.OptFlags.all_on(), layers=1)
    seqs = bt.SeqLengths.of([3, 8], 8)
    w = None
    with pytest.raises(bt.ShapeError, match="rows"):
        bt.forward(w, seqs, np.zeros((15, 768), np.float32), cfg)
    with pytest.raises(bt.ShapeError, match="batch"):
        bt.forward(w, bt.SeqLengths.of([3], 8), np.zeros((8, 768), np.float32), cfg)
    with pytest.raises(bt.ShapeError, match="columns"):
        bt.forward(w, seqs, np.zeros((16, 64), np.float32), cfg)


def test_flop_model_matches_oracle():
    """The exact FLOP model bench --check compares the instrumented counts
    with (flops.count, reference flops.py:72-110) agrees with the oracle's
    restatement for the packed and the padded variants."""
    from paper_2210_03052_b200 import flops

    lens = orc.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6)
    seqs = bt.SeqLengths.of(lens, 256)
    cfg = bt.preset_config("bert_base", 16, 256, bt.OptFlags.all_on())
    assert flops.count(cfg, seqs, "zero_padding_fused_mha").exact == orc.exact_flops(lens, 768)
    assert flops.count(cfg, seqs, "baseline").exact == orc.exact_flops(lens, 768, fused=False, max_seq_len=256)


def test_harness_generators_match_reference(golden):
    from paper_2210_03052_b200 import harness

    g = golden("generators")
    for tag, (bs, mx) in {"c1": (16, 128), "c2": (16, 256), "c3": (16, 512), "c5": (2048, 512)}.items():
        assert list(harness.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6).lengths) == g[f"{tag}_lengths"].tolist()
    assert list(harness.gen_lengths(50, 77, "uniform", seed=4).lengths) == g["uniform_lengths"].tolist()
    seqs = bt.SeqLengths.of(g["input_lengths"].tolist(), 16)
    np.testing.assert_array_equal(harness.gen_input(seqs, 32, 2), g["input_x"])
    lens = g["c2_lengths"].tolist()
    assert harness.layer_flops(lens, 768) == {k: int(g[f"flops_c2_{k}"]) for k in
                                              ("gemm0", "mha", "gemm1", "gemm2", "gemm3")}


def test_token_balanced_partition():
    from paper_2210_03052_b200 import harness
    from paper_2210_03052_b200.partition import imbalance, token_balanced_partition

    lens = harness.gen_lengths(2048, 512, "fixed", seed=0, alpha=0.6).lengths
    for n in (1, 2, 4, 8):
        sh = token_balanced_partition(lens, n, 1024)
        assert sh[0].start == 0 and sh[-1].stop == 2048
        assert all(a.stop == b.start for a, b in zip(sh, sh[1:]))
        assert sum(s.tokens for s in sh) == sum(lens)
        assert imbalance(sh) < 1.01
    with pytest.raises(ValueError):
        token_balanced_partition([3, 4], 3)


def test_host_io_chunk_bounds():
    """Sequence ranges of the host-I/O pipeline (BertEncoderB200.chunk_bounds):
    contiguous, non-empty, covering every sequence once, at most the asked
    count, cut near the token-balanced targets."""
    from paper_2210_03052_b200 import harness
    from paper_2210_03052_b200.encoder import BertEncoderB200

    lens = harness.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6).lengths
    for chunks in (1, 2, 3, 4, 16, 40, [0.3, 0.7], [0.2, 0.6, 0.2]):
        b = BertEncoderB200.chunk_bounds(lens, chunks)
        n = chunks if isinstance(chunks, int) else len(chunks)
        assert 1 <= len(b) <= min(n, len(lens))
        assert b[0][0] == 0 and b[-1][1] == len(lens)
        assert all(b0 < b1 for b0, b1 in b) and all(b[i][1] == b[i + 1][0] for i in range(len(b) - 1))
    two = BertEncoderB200.chunk_bounds(lens, 2)
    first = sum(lens[two[0][0]:two[0][1]])
    assert abs(first - sum(lens) / 2) <= max(lens)  # the boundary nearest the half-way token count
    assert BertEncoderB200.chunk_bounds([7], 3) == [(0, 1)]
