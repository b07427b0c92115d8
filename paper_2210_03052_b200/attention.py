"""Fused variable-length multi-head attention on the B200 (reference
attention.py:1-314).

``dispatch_mha`` keeps the reference's routing rule -- the tile-resident
short kernel iff ``plan.max_seq_len <= cutoff`` (default 384), else the
long kernel over per-sequence problem sizes -- and its API.  The kernels
(``csrc/mha_sm100.cu``) read one packed ``[T, 3k]`` bf16 QKV tensor with the
Q/K/V biases already added, so the operator-level entry points here build
that tensor on the device (one bias-add pass per operand) and call
``bt_mha_varlen``.  In the encoder the QKV GEMM epilogue produces it directly.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError
from .packing import PackingPlan, ensure_plan
from .tensor import FlopCounter, Tensor, host_array, is_device, rows_cols

DEFAULT_CUTOFF = 384
DEFAULT_SPLIT_SEQ_LEN = 32
SHORT_MAX_KEYS = 384   # on-chip capacity of the short kernel (TMEM: 384 S + 64 O columns)


@dataclass
class AttentionInput:
    """Q, K, V, their biases, the plan and head geometry (reference
    attention.py:37-90)."""

    q: object
    k: object
    v: object
    q_bias: object
    k_bias: object
    v_bias: object
    plan: PackingPlan
    head_num: int
    head_size: int

    def __post_init__(self):
        hidden = self.head_num * self.head_size
        for name, t in (("q", self.q), ("k", self.k), ("v", self.v)):
            if rows_cols(t)[1] != hidden:
                raise ShapeError(f"{name} has {rows_cols(t)[1]} columns, expected head_num * head_size = {hidden}")
        for name, b in (("q_bias", self.q_bias), ("k_bias", self.k_bias), ("v_bias", self.v_bias)):
            shape = tuple(b.shape) if is_device(b) else np.shape(b)
            if shape != (hidden,):
                raise ShapeError(f"{name} must have length {hidden}")
        if not (rows_cols(self.q)[0] == rows_cols(self.k)[0] == rows_cols(self.v)[0]):
            raise ShapeError("q, k, v must have the same number of rows")

    @property
    def hidden_dim(self) -> int:
        return self.head_num * self.head_size

    @property
    def scale(self) -> float:
        return 1.0 / math.sqrt(self.head_size)

    def require_packed(self, op: str) -> None:
        if rows_cols(self.q)[0] != self.plan.valid_word_cnt:
            raise ShapeError(f"{op} expects packed layout ({self.plan.valid_word_cnt} rows), got {rows_cols(self.q)[0]}")

    def require_padded(self, op: str) -> None:
        if rows_cols(self.q)[0] != self.plan.padded_rows:
            raise ShapeError(f"{op} expects padded layout ({self.plan.padded_rows} rows), got {rows_cols(self.q)[0]}")


def mha_device(qkv_bf16, plan: PackingPlan, head_num: int, head_size: int, *, cutoff: int = DEFAULT_CUTOFF,
               split_seq_len: int = DEFAULT_SPLIT_SEQ_LEN, path: int = 0, out=None):
    """Fused MHA over a packed, biased QKV tensor [T, 3k] (bf16, device)."""
    torch = _lib.require_device()
    T = plan.valid_word_cnt
    hidden = head_num * head_size
    if tuple(qkv_bf16.shape) != (T, 3 * hidden):
        raise ShapeError(f"qkv must be [{T}, {3 * hidden}], got {tuple(qkv_bf16.shape)}")
    if out is None:
        out = torch.empty((T, hidden), dtype=torch.bfloat16, device=qkv_bf16.device)
    if path == 0:
        _lib.call("bt_mha_varlen", qkv_bf16.data_ptr(), plan.seq_starts_dev.data_ptr(), plan.batch_size,
                  plan.max_seq_len, head_num, head_size, int(cutoff), int(split_seq_len), out.data_ptr(), T,
                  _lib.stream_ptr())
    else:
        _lib.call("bt_mha_varlen_path", qkv_bf16.data_ptr(), plan.seq_starts_dev.data_ptr(), plan.batch_size,
                  plan.max_seq_len, head_num, head_size, out.data_ptr(), T, int(path), _lib.stream_ptr())
    return out


def _qkv_device(inp: AttentionInput):
    """Concatenate Q|K|V with their biases added into one bf16 [T, 3k] tensor."""
    torch = _lib.require_device()
    from .fusion import bias_act_device

    T, hid = rows_cols(inp.q)
    qkv = torch.empty((T, 3 * hid), dtype=torch.bfloat16, device="cuda")
    for i, (t, b) in enumerate(((inp.q, inp.q_bias), (inp.k, inp.k_bias), (inp.v, inp.v_bias))):
        src = t.to(torch.float32).contiguous() if is_device(t) else torch.from_numpy(host_array(t)).to("cuda")
        bias = b.to(torch.float32).contiguous() if is_device(b) else torch.from_numpy(
            np.ascontiguousarray(np.asarray(b, np.float32))).to("cuda")
        bias_act_device(src, bias, 0, out=qkv[:, i * hid:(i + 1) * hid])
    return qkv


def _run(inp: AttentionInput, op: str, path: int, cutoff: int, split_seq_len: int, counter):
    inp.plan = ensure_plan(inp.plan)
    inp.require_packed(op)
    qkv = _qkv_device(inp)
    if counter is None:
        out = mha_device(qkv, inp.plan, inp.head_num, inp.head_size, cutoff=cutoff, split_seq_len=split_seq_len,
                         path=path)
    else:
        # instrumented: the kernel's tiles count the work they did (instrument.py)
        from .instrument import LaunchFlops

        with LaunchFlops() as lf:
            out = mha_device(qkv, inp.plan, inp.head_num, inp.head_size, cutoff=cutoff,
                             split_seq_len=split_seq_len, path=path)
        counter.add("mha", lf.counts["mha"])
    return out.float() if is_device(inp.q) else Tensor(out.float().cpu().numpy())


def mha_fused_short(inp: AttentionInput, split_seq_len: int = DEFAULT_SPLIT_SEQ_LEN, *, cutoff: int = DEFAULT_CUTOFF,
                    workers: int = 1, counter: FlopCounter | None = None):
    """Tile-resident short-sequence path (reference attention.py:177-237)."""
    plan = ensure_plan(inp.plan)
    mx = plan.max_seq_len
    if mx > cutoff:
        raise ShapeError(f"max_seq_len {mx} exceeds the short-path cutoff {cutoff}")
    if split_seq_len < 1:
        raise ShapeError(f"split_seq_len must be >= 1, got {split_seq_len}")
    if mx > SHORT_MAX_KEYS:
        raise ShapeError(f"the on-chip short kernel holds at most {SHORT_MAX_KEYS} keys, max_seq_len is {mx}")
    return _run(inp, "mha_fused_short", 1, cutoff, split_seq_len, counter)


def mha_fused_long(inp: AttentionInput, workers: int = 1, *, tile_m: int = 128, tile_n: int = 128,
                   counter: FlopCounter | None = None):
    """Grouped long-sequence path (reference attention.py:240-296)."""
    if tile_m < 1 or tile_n < 1:
        raise ShapeError(f"tile sizes must be >= 1, got ({tile_m}, {tile_n})")
    return _run(inp, "mha_fused_long", 2, DEFAULT_CUTOFF, DEFAULT_SPLIT_SEQ_LEN, counter)


def dispatch_mha(inp: AttentionInput, *, cutoff: int = DEFAULT_CUTOFF, split_seq_len: int = DEFAULT_SPLIT_SEQ_LEN,
                 workers: int = 1, tile_m: int = 128, tile_n: int = 128, counter: FlopCounter | None = None):
    """Short path iff max_seq_len <= cutoff, else the long path (reference
    attention.py:299-314)."""
    plan = ensure_plan(inp.plan)
    if plan.max_seq_len <= cutoff:
        if split_seq_len < 1:
            raise ShapeError(f"split_seq_len must be >= 1, got {split_seq_len}")
        return _run(inp, "mha_fused_short", 0, cutoff, split_seq_len, counter)
    return mha_fused_long(inp, workers, tile_m=tile_m, tile_n=tile_n, counter=counter)
