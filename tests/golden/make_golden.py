"""Freeze golden vectors from the REFERENCE implementation (packbert 0.1.0).

Run in the build container, where /root/reference exists:

    python tests/golden/make_golden.py

It imports the unmodified reference from /root/reference/pkg/src, runs it on
seeded inputs and writes small ``.npz`` fixtures next to this script.  The GPU
box never runs this script (the reference does not travel); tests there read
the committed fixtures.  The fixtures pin ``oracle/packbert_np.py`` (checked in
``tests/test_oracle_golden.py``), which in turn is the checker for the CUDA
path at sizes where a fixture would be too large.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
sys.path.insert(0, str(HERE.parents[1]))

import packbert as pb  # noqa: E402  (the reference)
from packbert import attention as pba  # noqa: E402
from packbert import bench as pbb  # noqa: E402
from packbert import encoder as pbe  # noqa: E402
from packbert import fusion as pbf  # noqa: E402
from packbert import packing as pbp  # noqa: E402

from oracle import packbert_np as orc  # noqa: E402  (only for the stress weight recipe)


def _save(name: str, **arrays):
    path = HERE / f"{name}.npz"
    np.savez_compressed(path, **arrays)
    print(f"wrote {path.name}: {path.stat().st_size / 1024:.1f} KiB, keys={sorted(arrays)}")


def _ref_weights_from_dicts(dicts, cfg):
    layers = []
    for d in dicts:
        layers.append(pbe._layer_from_arrays({k: np.asarray(v, np.float32) for k, v in d.items()}))
    return pbe.EncoderWeights(layers=layers, shared=cfg.share_layer_weights)


def packing_cases():
    out = {}
    kats = {"fig4": ([2, 4, 5], 5), "ones": ([1, 1], 4), "dense": ([5, 5, 5], 5), "single": ([1], 8)}
    for tag, (lens, mx) in kats.items():
        plan = pbp.plan_for_lengths(pbp.SeqLengths.of(lens, mx))
        out[f"{tag}_lengths"] = np.asarray(lens, np.int64)
        out[f"{tag}_mx"] = np.int64(mx)
        out[f"{tag}_offsets"] = np.asarray(plan.offsets)
        out[f"{tag}_seq_starts"] = np.asarray(plan.seq_starts)
    # Fig. 4 unpack: packed row value = row index; padded zero rows {2,3,4,9}
    plan = pbp.plan_for_lengths(pbp.SeqLengths.of([2, 4, 5], 5))
    packed = pb.Tensor(np.repeat(np.arange(11, dtype=np.float32)[:, None] + 1.0, 3, axis=1))
    out["fig4_unpacked"] = pbp.unpack(pbp.PackedBatch(packed, plan), 5).array
    # random plans + pack/unpack round trip
    for tag, (bs, mx, seed) in {"r1": (37, 100, 3), "r2": (64, 1024, 7), "r3": (300, 17, 11)}.items():
        seqs = pbb.gen_lengths(bs, mx, "uniform", seed)
        plan = pbp.plan_for_lengths(seqs)
        out[f"{tag}_lengths"] = np.asarray(seqs.lengths, np.int64)
        out[f"{tag}_mx"] = np.int64(mx)
        out[f"{tag}_offsets"] = np.asarray(plan.offsets)
        out[f"{tag}_seq_starts"] = np.asarray(plan.seq_starts)
    seqs = pbb.gen_lengths(9, 40, "uniform", 5)
    plan = pbp.plan_for_lengths(seqs)
    x = pbb._gen_input(seqs, 24, 5)
    x.array[~pbp.build_mask(seqs).reshape(-1).astype(bool)] = 7.0  # non-zero padding
    packed = pbp.pack(x, plan)
    out["pk_lengths"] = np.asarray(seqs.lengths, np.int64)
    out["pk_padded"] = x.array
    out["pk_packed"] = packed.tokens.array
    out["pk_unpacked"] = pbp.unpack(packed, 40).array
    _save("packing", **out)


def generator_cases():
    out = {}
    cfgs = {"c1": (16, 128), "c2": (16, 256), "c3": (16, 512), "c5": (2048, 512)}
    for tag, (bs, mx) in cfgs.items():
        seqs = pbb.gen_lengths(bs, mx, "fixed", seed=0, alpha=0.6)
        out[f"{tag}_lengths"] = np.asarray(seqs.lengths, np.int64)
    out["uniform_lengths"] = np.asarray(pbb.gen_lengths(50, 77, "uniform", seed=4).lengths, np.int64)
    seqs = pbb.gen_lengths(4, 16, "fixed", seed=2, alpha=0.5)
    out["input_lengths"] = np.asarray(seqs.lengths, np.int64)
    out["input_x"] = pbb._gen_input(seqs, 32, 2).array
    cfg = pbe.ModelConfig(layers=2, head_num=2, head_size=8, max_seq_len=16, batch_size=4)
    w = pbe.init_weights(cfg, seed=3)
    for li, layer in enumerate(w.layers):
        for name, arr in pbe._layer_arrays(layer).items():
            out[f"w{li}_{name}"] = np.asarray(arr)
    # flop model (Table II) for C2
    c2 = pbe.preset_config("bert_base", 16, 256, pbe.OptFlags.all_on())
    rep = pb.count(c2, pbb.gen_lengths(16, 256, "fixed", seed=0, alpha=0.6), "zero_padding_fused_mha")
    for key, val in rep.exact.items():
        out[f"flops_c2_{key}"] = np.int64(val)
    _save("generators", **out)


def fusion_cases():
    rng = np.random.default_rng(21)
    out = {}
    out["gelu_in"] = np.linspace(-6, 6, 97, dtype=np.float32)
    out["gelu_out"] = np.asarray(pbf.gelu(out["gelu_in"]), np.float32)
    x = rng.standard_normal((33, 768)).astype(np.float32)
    r = rng.standard_normal((33, 768)).astype(np.float32)
    b = rng.standard_normal(768).astype(np.float32) * 0.1
    g = rng.standard_normal(768).astype(np.float32)
    be = rng.standard_normal(768).astype(np.float32)
    y = pbf.add_bias_residual_layernorm(pb.Tensor(x), pb.Tensor(r), b, pbf.LayernormParams(g, be))
    out.update(ln_x=x, ln_r=r, ln_b=b, ln_g=g, ln_beta=be, ln_y=y.array)
    kat = pbf.layernorm(pb.Tensor(np.array([[1, 2, 3]], np.float32)),
                        pbf.LayernormParams(np.ones(3, np.float32), np.zeros(3, np.float32)))
    out["ln_kat"] = kat.array
    _save("fusion", **out)


def attention_cases():
    out = {}
    for tag, (bs, mx, heads, seed) in {"short": (5, 64, 2, 1), "long": (3, 520, 2, 2),
                                       "cut384": (2, 384, 1, 3), "cut385": (2, 385, 1, 4)}.items():
        seqs = pbb.gen_lengths(bs, mx, "uniform", seed)
        plan = pbp.plan_for_lengths(seqs)
        T = plan.valid_word_cnt
        hid = heads * 64
        rng = np.random.default_rng(100 + seed)
        q, k, v = (rng.standard_normal((T, hid)).astype(np.float32) for _ in range(3))
        qkvb = (rng.standard_normal(3 * hid) * 0.1).astype(np.float32)
        inp = pba.AttentionInput(pb.Tensor(q), pb.Tensor(k), pb.Tensor(v), qkvb[:hid], qkvb[hid:2 * hid],
                                 qkvb[2 * hid:], plan, heads, 64)
        o = pba.dispatch_mha(inp)
        out.update({f"{tag}_lengths": np.asarray(seqs.lengths, np.int64), f"{tag}_mx": np.int64(mx),
                    f"{tag}_heads": np.int64(heads), f"{tag}_q": q, f"{tag}_k": k, f"{tag}_v": v,
                    f"{tag}_bias": qkvb, f"{tag}_out": o.array})
    _save("attention", **out)


def encoder_cases():
    out = {}
    cases = {
        # tag: (layers, heads, mx, bs, seed, flags, weights)
        "tiny": (2, 2, 48, 6, 0, pbe.OptFlags.all_on(), "init"),
        "tiny_long": (1, 2, 400, 3, 1, pbe.OptFlags.all_on(), "init"),
        "tiny_stress": (2, 2, 96, 5, 2, pbe.OptFlags.all_on(), "stress"),
        "tiny_stress_long": (1, 2, 450, 2, 3, pbe.OptFlags.all_on(), "stress"),
        "tiny_padded": (1, 2, 40, 4, 4, pbe.OptFlags(), "stress"),
        "tiny_rmpad": (1, 2, 40, 4, 4, pbe.OptFlags(True, True, True, False), "stress"),
    }
    for tag, (layers, heads, mx, bs, seed, flags, wkind) in cases.items():
        cfg = pbe.ModelConfig(layers=layers, head_num=heads, head_size=64, max_seq_len=mx,
                              batch_size=bs, flags=flags)
        seqs = pbb.gen_lengths(bs, mx, "fixed", seed=seed, alpha=0.6)
        x = pbb._gen_input(seqs, cfg.hidden_dim, seed)
        if wkind == "init":
            w = pbe.init_weights(cfg, seed)
        else:
            ocfg = orc.OracleConfig(layers, heads, 64, mx, bs)
            w = _ref_weights_from_dicts(orc.stress_weights(ocfg, seed), cfg)
        y = pbe.forward(w, seqs, x, cfg)
        out[f"{tag}_lengths"] = np.asarray(seqs.lengths, np.int64)
        out[f"{tag}_out"] = y.array
    # C1 itself (BERT-base, 1 layer, bs16, mx128, reference init): keep every 8th row
    cfg = pbe.preset_config("bert_base", 16, 128, pbe.OptFlags.all_on(), layers=1)
    seqs = pbb.gen_lengths(16, 128, "fixed", seed=0, alpha=0.6)
    x = pbb._gen_input(seqs, 768, 0)
    y = pbe.forward(pbe.init_weights(cfg, 0), seqs, x, cfg)
    out["c1_rows"] = np.arange(0, 16 * 128, 8)
    out["c1_out_sub"] = y.array[out["c1_rows"]]
    out["c1_out_norm"] = np.float64(np.linalg.norm(y.array.astype(np.float64)))
    _save("encoder", **out)


if __name__ == "__main__":
    packing_cases()
    generator_cases()
    fusion_cases()
    attention_cases()
    encoder_cases()
