"""Tensor carrier, FLOP accounting, and the GEMM entry points.

Mirrors the reference's numeric substrate (tensor.py:26-235): ``Tensor`` is
the same 2-D row-major float32 host matrix (``.array``), ``FlopCounter`` the
same 2-FLOPs-per-MAC accounting, ``EpilogueHook`` the same hook enumeration.
``gemm`` / ``batched_gemm`` run on the sm_100a tcgen05 kernel (bf16 operands,
fp32 accumulation): host tensors are uploaded, computed on the B200 and
returned as host ``Tensor``s; CUDA ``torch.Tensor`` operands stay on device.

Device operands are bf16 activations ``[M, K]`` and weights given in the
reference's ``[in, out]`` layout; the weight is transposed to ``[out, in]``
(K-major, the operand layout the tensor cores read) on upload.
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import Enum
from typing import Sequence

import numpy as np

from . import _lib
from .errors import ShapeError

DEFAULT_TILE_M = 64   # reference tensor.py:22-23 (accepted for API parity)
DEFAULT_TILE_N = 64


class Tensor:
    """A 2-D row-major float32 host matrix (reference tensor.py:26-63)."""

    __slots__ = ("array",)

    def __init__(self, array):
        if _is_torch(array):
            array = array.detach().float().cpu().numpy()
        arr = np.asarray(array, dtype=np.float32)
        if arr.ndim != 2:
            raise ShapeError(f"tensor must be 2-D, got shape {arr.shape}")
        self.array = np.ascontiguousarray(arr)

    @classmethod
    def zeros(cls, rows: int, cols: int) -> "Tensor":
        return cls(np.zeros((rows, cols), dtype=np.float32))

    @classmethod
    def random(cls, rows: int, cols: int, seed: int = 0, scale: float = 1.0) -> "Tensor":
        rng = np.random.default_rng(seed)
        return cls((rng.standard_normal((rows, cols)) * scale).astype(np.float32))

    @property
    def rows(self) -> int:
        return self.array.shape[0]

    @property
    def cols(self) -> int:
        return self.array.shape[1]

    @property
    def data(self) -> np.ndarray:
        return self.array.reshape(-1)

    def copy(self) -> "Tensor":
        return Tensor(self.array.copy())

    def __repr__(self) -> str:
        return f"Tensor({self.rows}x{self.cols})"


class EpilogueKind(str, Enum):
    NONE = "none"
    ADD_BIAS = "add_bias"
    ADD_BIAS_GELU = "add_bias_gelu"
    SCALE = "scale"
    SOFTMAX_PARTIAL_REDUCE = "softmax_partial_reduce"


@dataclass(frozen=True)
class EpilogueHook:
    """GEMM epilogue selector (reference tensor.py:66-106)."""

    kind: EpilogueKind = EpilogueKind.NONE
    bias: np.ndarray | None = None
    scale: float | None = None
    sink: object | None = None

    @classmethod
    def none(cls) -> "EpilogueHook":
        return cls()

    @classmethod
    def add_bias(cls, bias) -> "EpilogueHook":
        return cls(kind=EpilogueKind.ADD_BIAS, bias=np.asarray(bias, dtype=np.float32))

    @classmethod
    def add_bias_gelu(cls, bias) -> "EpilogueHook":
        return cls(kind=EpilogueKind.ADD_BIAS_GELU, bias=np.asarray(bias, dtype=np.float32))

    @classmethod
    def scale_by(cls, scale: float) -> "EpilogueHook":
        return cls(kind=EpilogueKind.SCALE, scale=float(scale))

    @classmethod
    def partial_reduce(cls, sink, scale: float | None = None) -> "EpilogueHook":
        return cls(kind=EpilogueKind.SOFTMAX_PARTIAL_REDUCE, sink=sink, scale=scale)


class FlopCounter:
    """Multiply-add accounting: 2 FLOPs per MAC (reference tensor.py:109-125)."""

    def __init__(self):
        self.counts: dict[str, int] = {}

    def add(self, key: str, flops: int) -> None:
        self.counts[key] = self.counts.get(key, 0) + int(flops)

    def get(self, key: str) -> int:
        return self.counts.get(key, 0)

    def total(self) -> int:
        return sum(self.counts.values())

    def as_dict(self) -> dict[str, int]:
        return dict(self.counts)


# ---------------------------------------------------------------------------
# host / device operand helpers
# ---------------------------------------------------------------------------

def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch") and hasattr(x, "is_cuda")


def is_device(x) -> bool:
    return _is_torch(x) and x.is_cuda


def host_array(x) -> np.ndarray:
    """fp32 2-D ndarray view of a reference/our Tensor, ndarray or torch tensor."""
    if hasattr(x, "array") and isinstance(getattr(x, "array"), np.ndarray):
        arr = x.array
    elif _is_torch(x):
        arr = x.detach().float().cpu().numpy()
    else:
        arr = np.asarray(x)
    arr = np.asarray(arr, dtype=np.float32)
    if arr.ndim != 2:
        raise ShapeError(f"tensor must be 2-D, got shape {arr.shape}")
    return np.ascontiguousarray(arr)


def rows_cols(x) -> tuple[int, int]:
    if is_device(x):
        if x.dim() != 2:
            raise ShapeError(f"tensor must be 2-D, got shape {tuple(x.shape)}")
        return int(x.shape[0]), int(x.shape[1])
    a = x.array if hasattr(x, "array") else np.asarray(x)
    if a.ndim != 2:
        raise ShapeError(f"tensor must be 2-D, got shape {a.shape}")
    return int(a.shape[0]), int(a.shape[1])


def to_device_bf16(x, torch=None):
    torch = torch or _lib.require_device()
    if is_device(x):
        return x.to(torch.bfloat16).contiguous()
    return torch.from_numpy(host_array(x)).to("cuda", non_blocking=False).to(torch.bfloat16).contiguous()


def to_device_f32(x, torch=None):
    torch = torch or _lib.require_device()
    if is_device(x):
        return x.to(torch.float32).contiguous()
    arr = x.array if hasattr(x, "array") else x
    return torch.from_numpy(np.ascontiguousarray(np.asarray(arr, np.float32))).to("cuda")


def weight_t_bf16(w, torch=None):
    """Reference [in, out] fp32 weight -> device bf16 [out, in] (K-major)."""
    torch = torch or _lib.require_device()
    if is_device(w):
        return w.t().to(torch.bfloat16).contiguous()
    return torch.from_numpy(np.ascontiguousarray(host_array(w).T)).to("cuda").to(torch.bfloat16)


def _ptr(t) -> int:
    return 0 if t is None else int(t.data_ptr())


def gemm_device(a_bf16, bt_bf16, bias_f32=None, residual_bf16=None, epilogue: int = _lib.EPI_NONE, out=None,
                bn: int | None = None):
    """C = epilogue(A @ Bt^T) on the tcgen05 kernel; all operands on device."""
    torch = _lib.require_device()
    M, K = a_bf16.shape
    N, K2 = bt_bf16.shape
    if K != K2:
        raise ShapeError(f"gemm dimension mismatch: ({M}x{K}) @ ({K2}x{N})")
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a_bf16.device)
    args = (_ptr(a_bf16), _ptr(bt_bf16), _ptr(bias_f32), _ptr(residual_bf16), _ptr(out), M, N, K, int(epilogue))
    if bn is None:
        _lib.call("bt_gemm", *args, _lib.stream_ptr())
    else:
        _lib.call("bt_gemm_bn", *args, int(bn), _lib.stream_ptr())
    return out


_EPI = {EpilogueKind.NONE: _lib.EPI_NONE, EpilogueKind.ADD_BIAS: _lib.EPI_BIAS,
        EpilogueKind.ADD_BIAS_GELU: _lib.EPI_BIAS_GELU}


def gemm(
    a,
    b,
    epilogue: EpilogueHook | None = None,
    tile_m: int = DEFAULT_TILE_M,
    tile_n: int = DEFAULT_TILE_N,
    *,
    counter: FlopCounter | None = None,
    key: str = "gemm",
):
    """``epilogue(a @ b)`` on the B200 tensor cores (reference tensor.py:177-200).

    Epilogues none / add_bias / add_bias_gelu run fused in the kernel; scale
    is applied in fp32 on the result.  ``tile_m``/``tile_n`` are validated and
    otherwise ignored (tile geometry is the kernel's; results never depend on
    it, as in the reference)."""
    if tile_m < 1 or tile_n < 1:
        raise ShapeError(f"tile sizes must be >= 1, got ({tile_m}, {tile_n})")
    am, ak = rows_cols(a)
    bk, bn = rows_cols(b)
    if ak != bk:
        raise ShapeError(f"gemm dimension mismatch: ({am}x{ak}) @ ({bk}x{bn})")
    hook = epilogue or EpilogueHook.none()
    if hook.kind == EpilogueKind.SOFTMAX_PARTIAL_REDUCE:
        raise ShapeError("softmax_partial_reduce is fused inside the MHA kernels; use dispatch_mha")
    if hook.kind in (EpilogueKind.ADD_BIAS, EpilogueKind.ADD_BIAS_GELU):
        if hook.bias is None or np.asarray(hook.bias).shape != (bn,):
            got = None if hook.bias is None else np.asarray(hook.bias).shape
            raise ShapeError(f"epilogue bias must have length {bn}, got {got}")
    torch = _lib.require_device()
    device_mode = is_device(a)
    A = to_device_bf16(a, torch)
    Bt = weight_t_bf16(b, torch)
    bias = None
    if hook.kind in _EPI and hook.kind != EpilogueKind.NONE:
        bias = to_device_f32(np.asarray(hook.bias, np.float32).reshape(-1), torch)
    # the kernel tiles K and N by 64: any other shape (the reference accepts
    # every shape) runs zero-padded on the device -- zero K columns add
    # nothing, padded N columns are sliced off
    kp, np_ = -(-ak // 64) * 64, -(-bn // 64) * 64
    if kp != ak:
        A = torch.nn.functional.pad(A, (0, kp - ak))
        Bt = torch.nn.functional.pad(Bt, (0, kp - ak))
    if np_ != bn:
        Bt = torch.nn.functional.pad(Bt, (0, 0, 0, np_ - bn))
        if bias is not None:
            bias = torch.nn.functional.pad(bias, (0, np_ - bn))
    C = gemm_device(A.contiguous(), Bt.contiguous(), bias, None, _EPI.get(hook.kind, _lib.EPI_NONE))
    out = C[:, :bn].float()
    if hook.kind == EpilogueKind.SCALE:
        out *= float(hook.scale)
    if counter is not None:
        counter.add(key, 2 * am * ak * bn)
    return out if device_mode else Tensor(out.cpu().numpy())


def batched_gemm(a_batch: Sequence, b_batch: Sequence, epilogue: EpilogueHook | None = None, *,
                 counter: FlopCounter | None = None, key: str = "gemm") -> list:
    """Identically shaped GEMMs (reference tensor.py:203-235).  When every A is
    the same operand (the QKV projection, encoder.py:358) the B matrices are
    concatenated along N and run as ONE kernel launch, then split."""
    if len(a_batch) != len(b_batch):
        raise ShapeError(f"batch counts differ: {len(a_batch)} vs {len(b_batch)}")
    if not a_batch:
        return []
    a_shape = rows_cols(a_batch[0])
    b_shape = rows_cols(b_batch[0])
    for i, (a, b) in enumerate(zip(a_batch, b_batch)):
        if rows_cols(a) != a_shape or rows_cols(b) != b_shape:
            ra, rb = rows_cols(a), rows_cols(b)
            raise ShapeError(
                f"batched GEMM requires identical shapes; batch {i} has ({ra[0]}x{ra[1]}) @ ({rb[0]}x{rb[1]}), "
                f"expected ({a_shape[0]}x{a_shape[1]}) @ ({b_shape[0]}x{b_shape[1]})")
    if all(a is a_batch[0] for a in a_batch) and (epilogue is None or epilogue.kind == EpilogueKind.NONE):
        wide = [host_array(b) if not is_device(b) else b for b in b_batch]
        if is_device(wide[0]):
            import torch as _t
            bcat = _t.cat(wide, dim=1)
        else:
            bcat = np.concatenate(wide, axis=1)
        c = gemm(a_batch[0], bcat)
        n = b_shape[1]
        if counter is not None:
            for _ in a_batch:
                counter.add(key, 2 * a_shape[0] * a_shape[1] * n)
        if is_device(c):
            return [c[:, i * n:(i + 1) * n].contiguous() for i in range(len(a_batch))]
        return [Tensor(c.array[:, i * n:(i + 1) * n]) for i in range(len(a_batch))]
    return [gemm(a, b, epilogue, counter=counter, key=key) for a, b in zip(a_batch, b_batch)]
