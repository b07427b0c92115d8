"""Padding-free batching on the B200: mask, prefix-sum plan, pack, unpack.

Mirrors the reference's packing module (packing.py:20-179) name for name.
The plan is computed on the device (``bt_plan_mask`` / ``bt_plan_lengths``:
warp-per-row mask reduction, exclusive prefix sum, offsets), pack/unpack are
16-byte-vectorised gather/scatter kernels.  Offsets and sequence starts are
int32 on the device and exposed as read-only int64 host arrays, bit-identical
to the reference's (``tests/test_gpu_packing.py``).

Host-side contract checks raise before any launch, with the reference's
exception types and messages (packing.py:27-36, 103-109, 143-147, 154-157).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ShapeError
from .tensor import Tensor, host_array, is_device, rows_cols


@dataclass(frozen=True)
class SeqLengths:
    """Token counts per sequence (reference packing.py:20-53)."""

    lengths: tuple[int, ...]
    max_seq_len: int

    def __post_init__(self):
        if not self.lengths:
            raise ShapeError("batch must contain at least one sequence")
        if self.max_seq_len < 1:
            raise ShapeError(f"max_seq_len must be >= 1, got {self.max_seq_len}")
        for i, n in enumerate(self.lengths):
            if not 1 <= n <= self.max_seq_len:
                raise ShapeError(f"sequence {i} has length {n}, expected 1..{self.max_seq_len}")

    @classmethod
    def of(cls, lengths, max_seq_len: int) -> "SeqLengths":
        return cls(tuple(int(n) for n in lengths), int(max_seq_len))

    @property
    def batch_size(self) -> int:
        return len(self.lengths)

    @property
    def total(self) -> int:
        return sum(self.lengths)

    @property
    def alpha(self) -> float:
        return self.total / (self.batch_size * self.max_seq_len)


def as_seq_lengths(seqs) -> SeqLengths:
    """Accept the reference's SeqLengths (duck-typed) or ours."""
    if isinstance(seqs, SeqLengths):
        return seqs
    return SeqLengths.of(seqs.lengths, seqs.max_seq_len)


def build_mask(seqs) -> np.ndarray:
    """Row i = lengths[i] ones then zeros, uint8 (reference packing.py:56-60)."""
    seqs = as_seq_lengths(seqs)
    cols = np.arange(seqs.max_seq_len)
    return (cols[None, :] < np.asarray(seqs.lengths)[:, None]).astype(np.uint8)


@dataclass(frozen=True, eq=False)
class PackingPlan:
    """Packed-row -> flat-padded-row mapping plus per-sequence starts.

    ``offsets_dev`` / ``seq_starts_dev`` / ``lengths_dev`` are device int32
    tensors consumed by the kernels; ``offsets`` / ``seq_starts`` are the
    reference's read-only int64 host arrays (fetched once, lazily)."""

    seqs: SeqLengths
    offsets_dev: object
    seq_starts_dev: object
    lengths_dev: object
    _host: dict = field(default_factory=dict, repr=False, compare=False)

    @property
    def offsets(self) -> np.ndarray:
        if "offsets" not in self._host:
            a = self.offsets_dev[: self.valid_word_cnt].cpu().numpy().astype(np.int64)
            a.setflags(write=False)
            self._host["offsets"] = a
        return self._host["offsets"]

    @property
    def seq_starts(self) -> np.ndarray:
        if "seq_starts" not in self._host:
            a = self.seq_starts_dev.cpu().numpy().astype(np.int64)
            a.setflags(write=False)
            self._host["seq_starts"] = a
        return self._host["seq_starts"]

    @property
    def valid_word_cnt(self) -> int:
        return self.seqs.total

    @property
    def batch_size(self) -> int:
        return self.seqs.batch_size

    @property
    def max_seq_len(self) -> int:
        return self.seqs.max_seq_len

    @property
    def padded_rows(self) -> int:
        return self.batch_size * self.max_seq_len

    @property
    def alpha(self) -> float:
        return self.valid_word_cnt / self.padded_rows

    def rows_of(self, batch_index: int) -> slice:
        start = int(np.sum(self.seqs.lengths[:batch_index]))
        return slice(start, start + self.seqs.lengths[batch_index])


def _validate_mask_host(mask: np.ndarray) -> None:
    if mask.ndim != 2:
        raise ShapeError(f"mask must be 2-D, got shape {mask.shape}")
    if not np.isin(mask, (0, 1)).all():
        raise ShapeError("mask entries must be 0 or 1")
    if (np.diff(mask.astype(np.int8), axis=1) > 0).any():
        raise ShapeError("mask rows must be a prefix of ones followed by zeros")


def compute_plan(mask) -> PackingPlan:
    """Plan from a 0/1 prefix-shaped mask via its prefix sum (reference
    packing.py:96-119), computed by the ``bt_plan_mask`` kernels.

    ``mask`` may be a host array (validated on the host first, as the
    reference does) or a CUDA uint8 tensor (validated on the device; one
    device->host read of the status word and T)."""
    torch = _lib.require_device()
    if is_device(mask):
        if mask.dim() != 2:
            raise ShapeError(f"mask must be 2-D, got shape {tuple(mask.shape)}")
        m = mask.to(torch.uint8).contiguous()
    else:
        host = np.asarray(mask)
        _validate_mask_host(host)
        m = torch.from_numpy(np.ascontiguousarray(host.astype(np.uint8))).to("cuda")
    bs, mx = int(m.shape[0]), int(m.shape[1])
    if bs < 1:
        raise ShapeError("batch must contain at least one sequence")
    lengths = torch.empty(bs, dtype=torch.int32, device="cuda")
    starts = torch.empty(bs + 1, dtype=torch.int32, device="cuda")
    offsets = torch.empty(bs * mx, dtype=torch.int32, device="cuda")
    misc = torch.zeros(2, dtype=torch.int32, device="cuda")  # [T, status]
    _lib.call("bt_plan_mask", m.data_ptr(), bs, mx, lengths.data_ptr(), starts.data_ptr(), offsets.data_ptr(),
              misc.data_ptr(), misc.data_ptr() + 4, _lib.stream_ptr())
    status = int(misc[1].item())
    if status & 1:
        raise ShapeError("mask entries must be 0 or 1")
    if status & 2:
        raise ShapeError("mask rows must be a prefix of ones followed by zeros")
    lens = lengths.cpu().numpy().tolist()
    seqs = SeqLengths.of(lens, mx)  # raises ShapeError for empty rows, like the reference
    return PackingPlan(seqs=seqs, offsets_dev=offsets, seq_starts_dev=starts, lengths_dev=lengths)


def plan_for_lengths(seqs) -> PackingPlan:
    """Plan straight from lengths (reference packing.py:122-123): the mask of
    a SeqLengths is prefix-shaped by construction, so the device skips the
    mask reduction and scans the lengths (``bt_plan_lengths``)."""
    torch = _lib.require_device()
    seqs = as_seq_lengths(seqs)
    lengths = torch.tensor(seqs.lengths, dtype=torch.int32).to("cuda")
    starts = torch.empty(seqs.batch_size + 1, dtype=torch.int32, device="cuda")
    offsets = torch.empty(max(seqs.total, 1), dtype=torch.int32, device="cuda")
    _lib.call("bt_plan_lengths", lengths.data_ptr(), seqs.batch_size, seqs.max_seq_len, starts.data_ptr(),
              offsets.data_ptr(), _lib.stream_ptr())
    return PackingPlan(seqs=seqs, offsets_dev=offsets, seq_starts_dev=starts, lengths_dev=lengths)


def ensure_plan(plan) -> PackingPlan:
    """Accept the reference's PackingPlan (host arrays) or ours."""
    if isinstance(plan, PackingPlan):
        return plan
    return plan_for_lengths(plan.seqs)


@dataclass(frozen=True)
class PackedBatch:
    """Valid token rows in contiguous order plus their plan (packing.py:126-138)."""

    tokens: object
    plan: PackingPlan

    def __post_init__(self):
        rows = rows_cols(self.tokens)[0]
        if rows != self.plan.valid_word_cnt:
            raise ShapeError(f"packed batch has {rows} rows, plan expects {self.plan.valid_word_cnt}")


def _dtype_code(t) -> int:
    import torch

    if t.dtype == torch.float32:
        return _lib.BT_F32
    if t.dtype == torch.bfloat16:
        return _lib.BT_BF16
    raise ShapeError(f"unsupported dtype {t.dtype}; expected float32 or bfloat16")


def pack_device(padded, plan: PackingPlan, out_dtype=None):
    """Device gather: padded CUDA tensor [bs*mx, k] -> packed [T, k]."""
    torch = _lib.require_device()
    out_dtype = out_dtype or padded.dtype
    T, k = plan.valid_word_cnt, int(padded.shape[1])
    out = torch.empty((T, k), dtype=out_dtype, device=padded.device)
    src = padded.contiguous()
    _lib.call("bt_pack", src.data_ptr(), _dtype_code(src), plan.offsets_dev.data_ptr(), T, k, out.data_ptr(),
              _dtype_code(out), _lib.stream_ptr())
    return out


def unpack_device(packed, plan: PackingPlan, out_dtype=None):
    """Device scatter with exact-zero padded rows: [T, k] -> [bs*mx, k]."""
    torch = _lib.require_device()
    out_dtype = out_dtype or torch.float32
    k = int(packed.shape[1])
    out = torch.empty((plan.padded_rows, k), dtype=out_dtype, device=packed.device)
    src = packed.contiguous()
    _lib.call("bt_unpack", src.data_ptr(), _dtype_code(src), plan.seq_starts_dev.data_ptr(), plan.batch_size,
              plan.max_seq_len, k, out.data_ptr(), _dtype_code(out), _lib.stream_ptr())
    return out


def pack(padded, plan) -> PackedBatch:
    """Gather the valid rows (reference packing.py:141-148).  Host input ->
    host fp32 tokens (bit-exact: the kernel moves fp32 words unchanged);
    CUDA input -> CUDA tokens of the same dtype."""
    plan = ensure_plan(plan)
    rows, cols = rows_cols(padded)
    if rows != plan.padded_rows:
        raise ShapeError(f"padded tensor has {rows} rows, plan expects "
                         f"{plan.batch_size} x {plan.max_seq_len} = {plan.padded_rows}")
    torch = _lib.require_device()
    if is_device(padded):
        return PackedBatch(tokens=pack_device(padded, plan), plan=plan)
    dev = torch.from_numpy(host_array(padded)).to("cuda")
    return PackedBatch(tokens=Tensor(pack_device(dev, plan).cpu().numpy()), plan=plan)


def unpack(packed: PackedBatch, max_seq_len: int):
    """Scatter back to padded positions, padded rows exactly zero (reference
    packing.py:151-160).  Returns a host fp32 Tensor for host tokens, a CUDA
    fp32 tensor for device tokens."""
    plan = ensure_plan(packed.plan)
    if max_seq_len != plan.max_seq_len:
        raise ShapeError(f"unpack max_seq_len {max_seq_len} does not match plan's {plan.max_seq_len}")
    torch = _lib.require_device()
    tok = packed.tokens
    if is_device(tok):
        return unpack_device(tok, plan)
    dev = torch.from_numpy(host_array(tok)).to("cuda")
    return Tensor(unpack_device(dev, plan).cpu().numpy())
