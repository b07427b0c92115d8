"""CPU-side checks of the C ABI boundary: the library is built for sm_100a,
loads without a GPU, and exports every symbol include/bt200.h declares."""

import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "bt200.h"
LIB = ROOT / "paper_2210_03052_b200" / "libbt200.so"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"BT_API\s+[\w\s\*]+?\b(bt_\w+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2210_03052_b200 import build, _lib

    build.build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for name in ("bt_plan_mask", "bt_plan_lengths", "bt_pack", "bt_unpack", "bt_gemm", "bt_mha_varlen",
                 "bt_ln_bias_residual", "bt_encoder_layer", "bt_encoder_forward", "bt_last_error"):
        assert name in syms


def test_library_exports_every_declared_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", str(LIB)], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (bt_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    # nothing else leaks out of the C ABI
    extra = sorted(s for s in exported if s not in declared_symbols())
    assert not extra, f"exported but not declared: {extra}"


def test_ctypes_signatures_cover_header(lib):
    from paper_2210_03052_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_symbols()
    assert lib.bt_version() >= 1


def test_sm100a_code_in_library(lib):
    r = subprocess.run(["cuobjdump", "-lelf", str(LIB)], capture_output=True, text=True)
    assert "sm_100a" in r.stdout
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "no tcgen05.mma in the library"
    assert "UTMALDG" in sass, "no TMA loads in the library"
    assert "LDTM" in sass, "no TMEM loads in the library"


def test_host_side_validation_without_gpu(lib):
    """Contract violations are rejected on the host before any CUDA call."""
    from paper_2210_03052_b200 import _lib

    assert lib.bt_gemm(None, None, None, None, None, 128, 100, 64, 0, None) == _lib.BT_ESHAPE
    assert "multiple of 64" in _lib.last_error()
    assert lib.bt_ln_bias_residual(None, None, None, None, None, 1e-12, None, 4, 12, None) == _lib.BT_ESHAPE
    assert lib.bt_mha_varlen(None, None, 1, 8, 1, 32, 384, 32, None, 8, None) == _lib.BT_ECONFIG
    assert lib.bt_pack(None, 0, None, 4, 0, None, 1, None) == _lib.BT_ESHAPE
