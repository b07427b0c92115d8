"""CPU oracle: a numpy restatement of the reference's padding-free encoder path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2210_03052_b200`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs use it, and only as the checker or
the timed CPU baseline -- never as a product path.

What it restates (reference = packbert 0.1.0 under /root/reference/pkg/src):

* packing    -- build_mask / compute_plan / pack / unpack      (packing.py:56-160)
* fusion     -- tanh-GELU, layernorm eps=1e-12, fused add-bias+residual+LN
                in the order (x + residual) + bias              (fusion.py:23-98)
* attention  -- padded baseline with -1e9 key masking          (attention.py:135-174)
                short fused path, per (seq, head) unit, q tiles (attention.py:177-237)
                long grouped path, 3 phases with float64 tile
                partials + full reduction                       (attention.py:104-122,240-296;
                                                                 grouped.py:190-251; tensor.py:128-173)
                dispatch rule max_seq_len <= cutoff             (attention.py:299-314)
* encoder    -- encoder_layer / forward, all OptFlags branches  (encoder.py:337-437)
* inputs     -- gen_lengths, _gen_input, init_weights           (bench.py:58-98,181-186;
                                                                 encoder.py:168-180)
* flops      -- exact per-layer FLOP model                      (flops.py:72-110)

Parity pinning: ``tests/golden/make_golden.py`` imports the reference itself
(in the build container, where /root/reference exists) and freezes its outputs
as ``tests/golden/*.npz``; ``tests/test_oracle_golden.py`` checks this module
against those fixtures bit-for-bit on the integer paths and to fp32 rounding
(<=1e-6 relative) on the float paths.

The arithmetic is numpy/OpenBLAS fp32 (plus the float64 softmax partials of
the long path), exactly like the reference, so timing this module on the host
is a faithful CPU baseline (``cpu_baseline.kind = "port"``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

MASK_VALUE = np.float32(-1e9)          # attention.py:34
DEFAULT_CUTOFF = 384                   # attention.py:32
DEFAULT_SPLIT_SEQ_LEN = 32             # attention.py:33
LN_EPS = 1e-12                         # fusion.py:42
WEIGHT_INIT_RANGE = 0.02               # encoder.py:34
_C_GELU = math.sqrt(2.0 / math.pi)     # fusion.py:19
_A_GELU = 0.044715                     # fusion.py:20


class OracleShapeError(ValueError):
    pass


# ----------------------------------------------------------------------------
# packing (packing.py)
# ----------------------------------------------------------------------------

def build_mask(lengths, max_seq_len: int) -> np.ndarray:
    """mask[b, j] = j < len[b] as uint8 (packing.py:56-60)."""
    lens = np.asarray(lengths, dtype=np.int64)
    return (np.arange(max_seq_len)[None, :] < lens[:, None]).astype(np.uint8)


def compute_plan(mask: np.ndarray):
    """(offsets int64[T], seq_starts int64[bs+1], lengths) (packing.py:96-119).

    Rows must be 0/1 and prefix-shaped; offsets are the flat indices of the
    ones in row-major order (the inverse of the inclusive prefix sum) and
    seq_starts the exclusive prefix sum of row sums.
    """
    m = np.asarray(mask)
    if m.ndim != 2:
        raise OracleShapeError("mask must be 2-D")
    if not np.isin(m, (0, 1)).all():
        raise OracleShapeError("mask entries must be 0 or 1")
    if (np.diff(m.astype(np.int8), axis=1) > 0).any():
        raise OracleShapeError("mask rows must be prefix-shaped")
    lengths = m.sum(axis=1, dtype=np.int64)
    offsets = np.flatnonzero(m.reshape(-1)).astype(np.int64)
    seq_starts = np.zeros(len(lengths) + 1, dtype=np.int64)
    np.cumsum(lengths, out=seq_starts[1:])
    return offsets, seq_starts, lengths


def pack(padded: np.ndarray, offsets: np.ndarray) -> np.ndarray:
    """Row gather packed[j] = padded[offsets[j]] (packing.py:141-148)."""
    return np.ascontiguousarray(np.asarray(padded, dtype=np.float32)[offsets])


def unpack(packed: np.ndarray, offsets: np.ndarray, padded_rows: int) -> np.ndarray:
    """Zero-filled row scatter (packing.py:151-160)."""
    out = np.zeros((padded_rows, packed.shape[1]), dtype=np.float32)
    out[offsets] = packed
    return out


# ----------------------------------------------------------------------------
# element-wise fusion (fusion.py)
# ----------------------------------------------------------------------------

def gelu(x):
    """0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))) (fusion.py:23-27)."""
    x = np.asarray(x, dtype=np.float32)
    return 0.5 * x * (1.0 + np.tanh(_C_GELU * (x + _A_GELU * x * x * x)))


def _ln_rows(z: np.ndarray, gamma, beta, eps: float = LN_EPS) -> np.ndarray:
    """Population-variance LN over rows (fusion.py:51-57)."""
    mu = z.mean(axis=1, keepdims=True)
    c = z - mu
    var = (c * c).mean(axis=1, keepdims=True)
    return gamma * (c / np.sqrt(var + np.float32(eps))) + beta


def add_bias_residual_layernorm(x, residual, bias, gamma, beta, eps: float = LN_EPS):
    """LN((x + residual) + bias) (fusion.py:79-98)."""
    z = (np.asarray(x, np.float32) + np.asarray(residual, np.float32)) + np.asarray(bias, np.float32)
    return _ln_rows(z, np.asarray(gamma, np.float32), np.asarray(beta, np.float32), eps)


def layernorm(x, gamma, beta, eps: float = LN_EPS):
    return _ln_rows(np.asarray(x, np.float32), np.asarray(gamma, np.float32), np.asarray(beta, np.float32), eps)


# ----------------------------------------------------------------------------
# attention (attention.py, grouped.py, tensor.py)
# ----------------------------------------------------------------------------

def _split_bias(qkv_bias: np.ndarray, hidden: int):
    b = np.asarray(qkv_bias, dtype=np.float32)
    return b[:hidden], b[hidden:2 * hidden], b[2 * hidden:]


def mha_padded(q, k, v, qb, kb, vb, lengths, max_seq_len, head_num, head_size):
    """Padded oracle: -1e9 on padded keys, padded query rows zeroed
    (attention.py:135-174, zero_pad_softmax=False branch)."""
    bs = len(lengths)
    mx = max_seq_len
    hid = head_num * head_size
    scale = np.float32(1.0 / math.sqrt(head_size))

    def heads(t, b):
        a = np.asarray(t, np.float32).reshape(bs, mx, head_num, head_size).transpose(0, 2, 1, 3)
        return a + np.asarray(b, np.float32).reshape(head_num, 1, head_size)

    q4, k4, v4 = heads(q, qb), heads(k, kb), heads(v, vb)
    s = (q4 @ k4.swapaxes(-1, -2)) * scale
    lens = np.asarray(lengths)
    kpad = np.arange(mx)[None, :] >= lens[:, None]
    s = np.where(kpad[:, None, None, :], MASK_VALUE, s)
    s = np.exp(s - s.max(axis=-1, keepdims=True))
    p = s / s.sum(axis=-1, keepdims=True)
    o = np.ascontiguousarray((p @ v4).transpose(0, 2, 1, 3)).reshape(bs * mx, hid)
    o[kpad.reshape(-1)] = 0.0
    return o


def mha_short(q, k, v, qb, kb, vb, seq_starts, head_num, head_size, split_seq_len=DEFAULT_SPLIT_SEQ_LEN):
    """Tile-resident short path: per (seq, head), q tiles of split_seq_len rows,
    row softmax held whole (attention.py:177-237)."""
    T = q.shape[0]
    hid = head_num * head_size
    scale = np.float32(1.0 / math.sqrt(head_size))
    out = np.zeros((T, hid), dtype=np.float32)
    for b in range(len(seq_starts) - 1):
        r0, r1 = int(seq_starts[b]), int(seq_starts[b + 1])
        for h in range(head_num):
            c = slice(h * head_size, (h + 1) * head_size)
            kk = k[r0:r1, c] + kb[c]
            vv = v[r0:r1, c] + vb[c]
            for t in range(r0, r1, split_seq_len):
                te = min(t + split_seq_len, r1)
                s = ((q[t:te, c] + qb[c]) @ kk.T) * scale
                e = np.exp(s - s.max(axis=1, keepdims=True))
                e /= e.sum(axis=1, keepdims=True)
                out[t:te, c] = e @ vv
    return out


def mha_long(q, k, v, qb, kb, vb, seq_starts, head_num, head_size, tile_n=128):
    """Grouped long path (attention.py:240-296): phase 1 scaled logits with
    per-128-column float64 (max, sum exp) partials (tensor.py:128-138,166-173),
    full reduction (attention.py:104-122), phase 2 exp(x-max)/sum applied on
    operand load in fp32 (grouped.py:202-206) times V."""
    T = q.shape[0]
    hid = head_num * head_size
    scale = np.float32(1.0 / math.sqrt(head_size))
    out = np.zeros((T, hid), dtype=np.float32)
    for b in range(len(seq_starts) - 1):
        r0, r1 = int(seq_starts[b]), int(seq_starts[b + 1])
        n = r1 - r0
        for h in range(head_num):
            c = slice(h * head_size, (h + 1) * head_size)
            qq = q[r0:r1, c] + qb[c]
            kk = np.ascontiguousarray((k[r0:r1, c] + kb[c]).T)
            vv = v[r0:r1, c] + vb[c]
            logits = qq @ kk
            logits *= scale
            ntile = math.ceil(n / tile_n)
            pm = np.empty((n, ntile))
            ps = np.empty((n, ntile))
            for j in range(ntile):
                blk = logits[:, j * tile_n:(j + 1) * tile_n].astype(np.float64)
                pm[:, j] = blk.max(axis=1)
                ps[:, j] = np.exp(blk - pm[:, j:j + 1]).sum(axis=1)
            gmax = pm.max(axis=1)
            gsum = (ps * np.exp(pm - gmax[:, None])).sum(axis=1)
            a = np.exp(logits - gmax.astype(np.float32)[:, None]) / gsum.astype(np.float32)[:, None]
            out[r0:r1, c] = a @ vv
    return out


def dispatch_mha(q, k, v, qkv_bias, seq_starts, max_seq_len, head_num, head_size,
                 cutoff=DEFAULT_CUTOFF, split_seq_len=DEFAULT_SPLIT_SEQ_LEN):
    """short iff max_seq_len <= cutoff (attention.py:299-314)."""
    hid = head_num * head_size
    qb, kb, vb = _split_bias(qkv_bias, hid)
    if max_seq_len <= cutoff:
        return mha_short(q, k, v, qb, kb, vb, seq_starts, head_num, head_size, split_seq_len)
    return mha_long(q, k, v, qb, kb, vb, seq_starts, head_num, head_size)


# ----------------------------------------------------------------------------
# model (encoder.py)
# ----------------------------------------------------------------------------

TENSOR_ORDER = (
    ("qkv_weight", lambda h, f: (h, 3 * h)),
    ("qkv_bias", lambda h, f: (3 * h,)),
    ("attn_out_weight", lambda h, f: (h, h)),
    ("attn_out_bias", lambda h, f: (h,)),
    ("ffn_w1", lambda h, f: (h, f)),
    ("ffn_b1", lambda h, f: (f,)),
    ("ffn_w2", lambda h, f: (f, h)),
    ("ffn_b2", lambda h, f: (h,)),
    ("ln0_gamma", lambda h, f: (h,)),
    ("ln0_beta", lambda h, f: (h,)),
    ("ln1_gamma", lambda h, f: (h,)),
    ("ln1_beta", lambda h, f: (h,)),
)  # declaration order of encoder.py:134-150


@dataclass
class OracleConfig:
    layers: int
    head_num: int
    head_size: int
    max_seq_len: int
    batch_size: int
    ffn_scale: int = 4
    cutoff: int = DEFAULT_CUTOFF
    split_seq_len: int = DEFAULT_SPLIT_SEQ_LEN
    share_layer_weights: bool = False

    @property
    def hidden(self) -> int:
        return self.head_num * self.head_size


def init_weights(cfg: OracleConfig, seed: int = 0) -> list[dict]:
    """U(-0.02, 0.02) for every tensor, one draw per tensor in declaration
    order, one dict per stored layer (encoder.py:168-180)."""
    rng = np.random.default_rng(seed)
    h = cfg.hidden
    f = cfg.ffn_scale * h
    stored = 1 if cfg.share_layer_weights else cfg.layers
    out = []
    for _ in range(stored):
        out.append({name: rng.uniform(-WEIGHT_INIT_RANGE, WEIGHT_INIT_RANGE, shp(h, f)).astype(np.float32)
                    for name, shp in TENSOR_ORDER})
    return out


def stress_weights(cfg: OracleConfig, seed: int = 0) -> list[dict]:
    """A non-degenerate weight set: N(0, 1/fan_in)
    matrices, gamma = 1, beta = 0, biases N(0, 0.02).  Under the reference
    init the softmax is near-uniform from layer 2 on; this set exercises it."""
    rng = np.random.default_rng(10_000 + seed)
    h = cfg.hidden
    f = cfg.ffn_scale * h
    stored = 1 if cfg.share_layer_weights else cfg.layers
    out = []
    for _ in range(stored):
        d = {}
        for name, shp in TENSOR_ORDER:
            s = shp(h, f)
            if name.endswith("gamma"):
                d[name] = np.ones(s, np.float32)
            elif name.endswith("beta"):
                d[name] = np.zeros(s, np.float32)
            elif len(s) == 2:
                d[name] = (rng.standard_normal(s) / math.sqrt(s[0])).astype(np.float32)
            else:
                d[name] = (rng.standard_normal(s) * 0.02).astype(np.float32)
        out.append(d)
    return out


def layer_weights(weights: list[dict], cfg: OracleConfig, li: int) -> dict:
    """ALBERT sharing: stored layer 0 for every index (encoder.py:130-131)."""
    return weights[0] if cfg.share_layer_weights else weights[li]


def encoder_layer(x, w: dict, cfg: OracleConfig, seq_starts, lengths, *, fuse_layernorm=True,
                  fuse_bias_gelu=True, zero_padding=True, fused_mha=True):
    """One post-LN layer (encoder.py:337-408); x is packed iff zero_padding."""
    h = cfg.hidden
    x = np.asarray(x, np.float32)
    wqkv = w["qkv_weight"]
    q = x @ wqkv[:, :h]
    k = x @ wqkv[:, h:2 * h]
    v = x @ wqkv[:, 2 * h:]
    qb, kb, vb = _split_bias(w["qkv_bias"], h)
    mx = cfg.max_seq_len
    if not zero_padding:
        attn = mha_padded(q, k, v, qb, kb, vb, lengths, mx, cfg.head_num, cfg.head_size)
    elif not fused_mha:
        offs = np.concatenate([b * mx + np.arange(n) for b, n in enumerate(lengths)])
        pr = len(lengths) * mx
        pad = [unpack(t, offs, pr) for t in (q, k, v)]
        attn = pack(mha_padded(*pad, qb, kb, vb, lengths, mx, cfg.head_num, cfg.head_size), offs)
    else:
        attn = dispatch_mha(q, k, v, w["qkv_bias"], seq_starts, mx, cfg.head_num, cfg.head_size,
                            cfg.cutoff, cfg.split_seq_len)
    proj = attn @ w["attn_out_weight"]
    if fuse_layernorm:
        y0 = add_bias_residual_layernorm(proj, x, w["attn_out_bias"], w["ln0_gamma"], w["ln0_beta"])
    else:
        y0 = layernorm((proj + x) + w["attn_out_bias"], w["ln0_gamma"], w["ln0_beta"])
    h1 = y0 @ w["ffn_w1"]
    h1 = gelu(h1 + w["ffn_b1"])
    h2 = h1 @ w["ffn_w2"]
    if fuse_layernorm:
        return add_bias_residual_layernorm(h2, y0, w["ffn_b2"], w["ln1_gamma"], w["ln1_beta"])
    return layernorm((h2 + y0) + w["ffn_b2"], w["ln1_gamma"], w["ln1_beta"])


def forward(weights: list[dict], lengths, input_padded: np.ndarray, cfg: OracleConfig, **flags):
    """pack once -> L layers -> unpack once (encoder.py:411-437).  Default
    flags are OptFlags.all_on(), the north-star path."""
    zero_padding = flags.get("zero_padding", True)
    mask = build_mask(lengths, cfg.max_seq_len)
    offsets, seq_starts, lens = compute_plan(mask)
    x = pack(input_padded, offsets) if zero_padding else np.asarray(input_padded, np.float32)
    for li in range(cfg.layers):
        x = encoder_layer(x, layer_weights(weights, cfg, li), cfg, seq_starts, lens, **flags)
    if zero_padding:
        return unpack(x, offsets, len(lengths) * cfg.max_seq_len)
    return x


# ----------------------------------------------------------------------------
# synthetic inputs (bench.py) and FLOP model (flops.py)
# ----------------------------------------------------------------------------

def gen_lengths(batch_size: int, max_seq_len: int, mode: str = "uniform", seed: int = 0,
                alpha: float | None = None) -> list[int]:
    """Uniform draw in [1, mx]; 'fixed' then nudges round-robin (clamped to
    [1, mx]) until the total is round(alpha*mx*bs) (bench.py:58-98)."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, max_seq_len + 1, size=batch_size).astype(np.int64)
    if mode == "fixed":
        target = int(round(alpha * max_seq_len * batch_size))
        target = min(max(target, batch_size), batch_size * max_seq_len)
        gap = target - int(lens.sum())
        step = 0
        while gap:
            j = step % batch_size
            if gap > 0 and lens[j] < max_seq_len:
                lens[j] += 1
                gap -= 1
            elif gap < 0 and lens[j] > 1:
                lens[j] -= 1
                gap += 1
            step += 1
    elif mode != "uniform":
        raise OracleShapeError(f"unknown mode {mode}")
    return [int(n) for n in lens]


def gen_input(lengths, max_seq_len: int, hidden: int, seed: int = 0) -> np.ndarray:
    """N(0,1) fp32 from default_rng(seed + 1), padded rows zeroed (bench.py:181-186)."""
    rng = np.random.default_rng(seed + 1)
    x = rng.standard_normal((len(lengths) * max_seq_len, hidden)).astype(np.float32)
    x[~build_mask(lengths, max_seq_len).reshape(-1).astype(bool)] = 0.0
    return x


def exact_flops(lengths, hidden: int, ffn_scale: int = 4, fused: bool = True, max_seq_len: int | None = None) -> dict:
    """Per-layer exact counts (flops.py:72-110)."""
    T = int(sum(lengths))
    k = hidden
    ffn = 2 * ffn_scale
    if fused:
        mha = 4 * sum(n * n for n in lengths) * k
        m = T
    else:
        m = len(lengths) * max_seq_len
        mha = 4 * len(lengths) * max_seq_len * max_seq_len * k
    return {"gemm0": 6 * m * k * k, "mha": mha, "gemm1": 2 * m * k * k,
            "gemm2": ffn * m * k * k, "gemm3": ffn * m * k * k}
