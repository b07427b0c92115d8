"""Resident CTAs per SM of each MHA variant (bt_debug_mha_occupancy)."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2210_03052_b200 import _lib  # noqa: E402

_lib.require_device()
L = _lib.load()
for w, name in enumerate(["short/2", "short/3", "long", "multi-tile long"]):
    info = (C.c_int * 3)()
    n = L.bt_debug_mha_occupancy(w, info)
    print(f"{name:16s} CTAs/SM {n}  regs {info[0]}  static smem {info[1]}  max dyn smem {info[2]}")
