"""ctypes binding of the C ABI in ``include/bt200.h`` (``libbt200.so``).

The library is built in-tree (``paper_2210_03052_b200/libbt200.so``) by
``python -m paper_2210_03052_b200.build`` / ``__graft_entry__.build()``.
There is no CPU fallback: every compute entry point raises if the library or
a CUDA device is missing.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

from .errors import ConfigError, PackbertError, ShapeError

LIB_PATH = Path(__file__).resolve().parent / "libbt200.so"

BT_OK, BT_ESHAPE, BT_ECONFIG, BT_ECUDA, BT_EDATA = 0, -1, -2, -3, -4
BT_F32, BT_BF16 = 0, 1
EPI_NONE, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESIDUAL = 0, 1, 2, 3


class BtCudaError(PackbertError, RuntimeError):
    """A CUDA runtime/driver failure inside libbt200."""


class LayerWeightsC(C.Structure):
    _fields_ = [
        ("qkv_w", C.c_void_p), ("qkv_b", C.c_void_p),
        ("ao_w", C.c_void_p), ("ao_b", C.c_void_p),
        ("w1", C.c_void_p), ("b1", C.c_void_p),
        ("w2", C.c_void_p), ("b2", C.c_void_p),
        ("ln0_g", C.c_void_p), ("ln0_b", C.c_void_p),
        ("ln1_g", C.c_void_p), ("ln1_b", C.c_void_p),
        ("ln0_eps", C.c_float), ("ln1_eps", C.c_float),
    ]


class LayerCfgC(C.Structure):
    _fields_ = [("head_num", C.c_int), ("head_size", C.c_int), ("ffn_scale", C.c_int),
                ("max_seq_len", C.c_int), ("cutoff", C.c_int), ("split_seq_len", C.c_int)]


_P, _I, _F, _S, _SZ = C.c_void_p, C.c_int, C.c_float, C.c_void_p, C.c_size_t

# name -> (restype, argtypes); mirrors include/bt200.h one to one
SIGNATURES = {
    "bt_version": (_I, []),
    "bt_last_error": (C.c_char_p, []),
    "bt_launch_count": (C.c_longlong, []),
    "bt_num_sms": (_I, []),
    "bt_plan_mask": (_I, [_P, _I, _I, _P, _P, _P, _P, _P, _S]),
    "bt_plan_lengths": (_I, [_P, _I, _I, _P, _P, _S]),
    "bt_pack": (_I, [_P, _I, _P, _I, _I, _P, _I, _S]),
    "bt_unpack": (_I, [_P, _I, _P, _I, _I, _I, _P, _I, _S]),
    "bt_gemm": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _S]),
    "bt_mha_varlen": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _P, _I, _S]),
    "bt_mha_padded": (_I, [_P, _P, _I, _I, _I, _I, _P, _S]),
    "bt_ln_bias_residual": (_I, [_P, _P, _P, _P, _P, _F, _P, _I, _I, _S]),
    "bt_gemm_bias_residual_ln": (_I, [_P, _P, _P, _P, _P, _P, _F, _P, _I, _I, _I, _S]),
    "bt_fused_attn_out_ln": (_I, [_I, _I]),
    "bt_fused_ffn2_ln": (_I, [_I, _I, _I]),
    "bt_plan_sched": (_I, [_P, _I, _I, _P, _S]),
    "bt_plan_sched_bytes": (_SZ, [_I, _I]),
    "bt_plan_forward": (_I, [_P, _I, _I, _P, _P, _S]),
    "bt_pack_starts": (_I, [_P, _P, _I, _I, _I, _P, _S]),
    "bt_mha_varlen_sched": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _S]),
    "bt_forward_prologue": (_I, [_P, _I, _I, _I, _P, _P, _P, _P, _P, _P, _P, _I, _S]),
    "bt_ln_bias_residual_out": (_I, [_P, _P, _P, _P, _P, _F, _P, _P, _I, _I, _S]),
    "bt_one_launch_ends": (_I, [_I, _I]),
    "bt_layer_workspace_bytes": (_SZ, [C.POINTER(LayerCfgC), _I]),
    "bt_encoder_layer": (_I, [C.POINTER(LayerWeightsC), C.POINTER(LayerCfgC), _P, _I, _I, _P, _P, _SZ, _S]),
    "bt_forward_workspace_bytes": (_SZ, [C.POINTER(LayerCfgC), _I, _I]),
    "bt_encoder_forward": (_I, [C.POINTER(LayerWeightsC), _I, C.POINTER(LayerCfgC), _P, _I, _I, _P, _P, _P, _SZ,
                                _S]),
    "bt_encoder_forward_packed": (_I, [C.POINTER(LayerWeightsC), _I, C.POINTER(LayerCfgC), _P, _I, _I, _P, _P,
                                       _P, _SZ, _S]),
    "bt_copy_rows": (_I, [_P, _P, _P, _I, _I, C.c_longlong, _I, _S]),
    "bt_bias_act": (_I, [_P, _I, _I, _P, _P, _I, _I, _I, _I, _I, _S]),
    "bt_add": (_I, [_P, _P, _P, _I, C.c_longlong, _S]),
    "bt_gemm_bn": (_I, [_P, _P, _P, _P, _P, _I, _I, _I, _I, _I, _S]),
    "bt_debug_gemm_trace": (_I, [_P]),
    "bt_debug_gemm_mode": (_I, [_I]),
    "bt_debug_mha_trace": (_I, [_P]),
    "bt_debug_mha_qg": (_I, [_I]),
    "bt_debug_mha_list": (_I, [_I, _I]),
    "bt_debug_mha_seg": (_I, [_I]),
    "bt_debug_mha_occupancy": (_I, [_I, _P]),
    "bt_debug_forward_events": (_I, [_P, _I]),
    "bt_mha_varlen_path": (_I, [_P, _P, _I, _I, _I, _I, _P, _I, _I, _S]),
    "bt_flops_enable": (_I, [_P]),
    "bt_flops_read": (_I, [_P]),
    "bt_host_alloc": (_I, [_SZ, _I, C.POINTER(C.c_void_p)]),
    "bt_debug_mha64": (_I, [_I]),
    "bt_host_free": (_I, [_P]),
}

_lock = threading.Lock()
_lib = None


def load(build_if_missing: bool = False) -> C.CDLL:
    """Load libbt200.so (optionally building it first)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not LIB_PATH.exists():
            if build_if_missing:
                from . import build as _build

                _build.build()
            else:
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2210_03052_b200.build` "
                    "(there is no CPU fallback)")
        # BT_LIB_PATH: an A/B build variant (scripts/ab_build.sh); default the in-tree library
        path = os.environ.get("BT_LIB_PATH") or str(LIB_PATH)
        lib = C.CDLL(path, mode=os.RTLD_NOW | os.RTLD_GLOBAL)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def last_error() -> str:
    msg = load().bt_last_error()
    return msg.decode() if msg else ""


def check(rc: int, what: str = "") -> None:
    """Map a bt_* return code to the reference's exception types."""
    if rc == BT_OK:
        return
    msg = last_error() or what
    if rc == BT_ESHAPE or rc == BT_EDATA:
        raise ShapeError(msg)
    if rc == BT_ECONFIG:
        raise ConfigError(msg)
    raise BtCudaError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)


def launch_count() -> int:
    return int(load().bt_launch_count())


def require_device():
    """Return torch with a CUDA device, or raise (no CPU fallback)."""
    import torch

    if not torch.cuda.is_available():
        raise RuntimeError("paper_2210_03052_b200 needs a CUDA device (sm_100a B200); no CPU fallback exists")
    load()
    return torch


def stream_ptr(stream=None) -> int:
    import torch

    s = stream if stream is not None else torch.cuda.current_stream()
    return int(s.cuda_stream)
