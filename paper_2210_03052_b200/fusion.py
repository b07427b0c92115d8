"""Memory-bound operators and their fused forms on the B200 (reference
fusion.py:1-98).

``add_bias_residual_layernorm`` is the paper's one-round-trip fused kernel
(section III-C1): z = (x + residual) + bias, population-variance LN with
eps = 1e-12 by default, fp32 statistics in registers, bf16 activations in
HBM.  ``gelu`` / ``bias_gelu_epilogue`` / ``add`` / ``add_rowvec`` /
``layernorm`` are the unfused passes of the optimisation ladder.  Host
operands are uploaded and results returned as host ``Tensor``s; CUDA
operands stay on the device.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import ShapeError
from .tensor import Tensor, host_array, is_device, rows_cols

_SQRT_2_OVER_PI = math.sqrt(2.0 / math.pi)
_GELU_CUBIC = 0.044715


@dataclass(frozen=True)
class LayernormParams:
    """gamma / beta / eps (reference fusion.py:38-48)."""

    gamma: np.ndarray
    beta: np.ndarray
    eps: float = 1e-12

    def __post_init__(self):
        if self.eps <= 0:
            raise ShapeError(f"layernorm eps must be > 0, got {self.eps}")
        if np.shape(self.gamma) != np.shape(self.beta):
            raise ShapeError("gamma and beta must have the same shape")


def _dev(x, torch, dtype):
    if is_device(x):
        return x.to(dtype).contiguous()
    return torch.from_numpy(host_array(x)).to("cuda").to(dtype).contiguous()


def _vec_f32(v, torch):
    if v is None:
        return None
    if is_device(v):
        return v.to(torch.float32).contiguous().reshape(-1)
    return torch.from_numpy(np.ascontiguousarray(np.asarray(v, np.float32).reshape(-1))).to("cuda")


def _ret(out, device_mode: bool):
    return out if device_mode else Tensor(out.float().cpu().numpy())


def ln_device(x_bf16, residual_bf16, bias_f32, gamma_f32, beta_f32, eps: float, out=None):
    """Device LN((x + residual) + bias) on bf16 [T, k] tensors."""
    torch = _lib.require_device()
    T, k = int(x_bf16.shape[0]), int(x_bf16.shape[1])
    if out is None:
        out = torch.empty_like(x_bf16)
    p = lambda t: 0 if t is None else t.data_ptr()  # noqa: E731
    _lib.call("bt_ln_bias_residual", p(x_bf16), p(residual_bf16), p(bias_f32), p(gamma_f32), p(beta_f32),
              float(eps), out.data_ptr(), T, k, _lib.stream_ptr())
    return out


def gemm_ln_device(a_bf16, bt_bf16, bias_f32, residual_bf16, gamma_f32, beta_f32, eps: float, out=None):
    """Device LN((a bt^T + residual) + bias) in one fused kernel (bt_gemm_bias_residual_ln)."""
    torch = _lib.require_device()
    M, K = int(a_bf16.shape[0]), int(a_bf16.shape[1])
    N = int(bt_bf16.shape[0])
    if out is None:
        out = torch.empty((M, N), dtype=torch.bfloat16, device=a_bf16.device)
    _lib.call("bt_gemm_bias_residual_ln", a_bf16.data_ptr(), bt_bf16.data_ptr(), bias_f32.data_ptr(),
              residual_bf16.data_ptr(), gamma_f32.data_ptr(), beta_f32.data_ptr(), float(eps), out.data_ptr(), M, N,
              K, _lib.stream_ptr())
    return out


def add_bias_residual_layernorm(x, residual, bias, params: LayernormParams):
    """One-pass LN((x + residual) + bias) (reference fusion.py:79-98)."""
    xr, xc = rows_cols(x)
    rr, rc = rows_cols(residual)
    if (xr, xc) != (rr, rc):
        raise ShapeError(f"shape mismatch: ({xr}x{xc}) vs residual ({rr}x{rc})")
    if np.shape(bias) != (xc,) and not (is_device(bias) and tuple(bias.shape) == (xc,)):
        raise ShapeError(f"bias must have length {xc}, got {np.shape(bias)}")
    if np.shape(params.gamma) != (xc,) and not (is_device(params.gamma) and tuple(params.gamma.shape) == (xc,)):
        raise ShapeError(f"layernorm params sized {np.shape(params.gamma)}, tensor has {xc} cols")
    torch = _lib.require_device()
    out = ln_device(_dev(x, torch, torch.bfloat16), _dev(residual, torch, torch.bfloat16), _vec_f32(bias, torch),
                    _vec_f32(params.gamma, torch), _vec_f32(params.beta, torch), params.eps)
    return _ret(out, is_device(x))


def layernorm(x, params: LayernormParams):
    """Plain LN over rows (reference fusion.py:60-63)."""
    _, xc = rows_cols(x)
    if np.shape(params.gamma) != (xc,) and not (is_device(params.gamma) and tuple(params.gamma.shape) == (xc,)):
        raise ShapeError(f"layernorm params sized {np.shape(params.gamma)}, tensor has {xc} cols")
    torch = _lib.require_device()
    out = ln_device(_dev(x, torch, torch.bfloat16), None, None, _vec_f32(params.gamma, torch),
                    _vec_f32(params.beta, torch), params.eps)
    return _ret(out, is_device(x))


def bias_act_device(x, bias_f32, act: int, out=None, out_dtype=None):
    """out = act(x + bias) on device (act 0 = identity, 1 = tanh-GELU)."""
    torch = _lib.require_device()
    rows, cols = int(x.shape[0]), int(x.shape[1])
    out_dtype = out_dtype or x.dtype
    if out is None:
        out = torch.empty((rows, cols), dtype=out_dtype, device=x.device)
    code = lambda t: _lib.BT_F32 if t.dtype == torch.float32 else _lib.BT_BF16  # noqa: E731
    _lib.call("bt_bias_act", x.data_ptr(), code(x), int(x.stride(0)), 0 if bias_f32 is None else bias_f32.data_ptr(),
              out.data_ptr(), code(out), int(out.stride(0)), rows, cols, int(act), _lib.stream_ptr())
    return out


def add_device(x, y, out=None):
    torch = _lib.require_device()
    if out is None:
        out = torch.empty_like(x)
    code = _lib.BT_F32 if x.dtype == torch.float32 else _lib.BT_BF16
    _lib.call("bt_add", x.data_ptr(), y.data_ptr(), out.data_ptr(), code, x.numel(), _lib.stream_ptr())
    return out


def gelu(x):
    """tanh-approximation GELU (reference fusion.py:23-27) on the device.
    Accepts a 2-D tensor (host or CUDA); scalars / 1-D arrays are promoted."""
    torch = _lib.require_device()
    device_mode = is_device(x)
    if device_mode:
        t = x.to(torch.float32).contiguous()
        shape = t.shape
    else:
        a = np.asarray(x, np.float32)
        shape = a.shape
        t = torch.from_numpy(np.ascontiguousarray(a)).to("cuda")
    flat = t.reshape(1, -1)
    n = flat.shape[1]
    pad = (-n) % 8
    if pad:
        flat = torch.nn.functional.pad(flat, (0, pad))
    out = bias_act_device(flat.contiguous(), None, 1)[:, :n].reshape(shape)
    if device_mode:
        return out
    res = out.cpu().numpy()
    return res if res.ndim else np.float32(res)


def bias_gelu_epilogue(tile, bias):
    """gelu(tile + bias[col]) (reference fusion.py:30-35)."""
    _, cols = rows_cols(tile)
    if np.shape(bias) != (cols,) and not (is_device(bias) and tuple(bias.shape) == (cols,)):
        raise ShapeError(f"bias must have length {cols}, got {np.shape(bias)}")
    torch = _lib.require_device()
    out = bias_act_device(_dev(tile, torch, torch.float32), _vec_f32(bias, torch), 1)
    return out if is_device(tile) else out.cpu().numpy()


def add(x, y):
    """x + y (reference fusion.py:66-69)."""
    if rows_cols(x) != rows_cols(y):
        raise ShapeError(f"shape mismatch: {rows_cols(x)} + {rows_cols(y)}")
    torch = _lib.require_device()
    out = add_device(_dev(x, torch, torch.float32), _dev(y, torch, torch.float32))
    return _ret(out, is_device(x))


def add_rowvec(x, vec):
    """x + vec[col] (reference fusion.py:72-76)."""
    _, cols = rows_cols(x)
    if np.shape(vec) != (cols,) and not (is_device(vec) and tuple(vec.shape) == (cols,)):
        raise ShapeError(f"row vector must have length {cols}, got {np.shape(vec)}")
    torch = _lib.require_device()
    out = bias_act_device(_dev(x, torch, torch.float32), _vec_f32(vec, torch), 0)
    return _ret(out, is_device(x))
