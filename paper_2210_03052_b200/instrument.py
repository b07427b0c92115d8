"""Instrumented FLOP counting for ``counter=FlopCounter()`` (reference
tensor.py:198-199, attention.py:232-236: every kernel adds the work of the
call it just made).

Here the counts come from the launches themselves, not from a formula: the
C runtime adds 2*M*N*K of every GEMM it launches under the module key
(gemm0..gemm3), GEMMs launched from Python (the ladder rungs) add theirs
through :func:`count_gemm`, and every MHA tile (fused or padded kernel) adds
the FLOPs it computed to a device counter (``bt_flops_enable``).  The bench
``--check`` compares these with the exact model (flops.count) with zero
tolerance, as the reference bench does (bench.py:256-267)."""

from __future__ import annotations

import ctypes as C
import threading

from . import _lib

KEYS = ("gemm0", "gemm1", "gemm2", "gemm3")
_active = threading.local()
_lock = threading.Lock()  # the C-side counters are process-wide: one counting region at a time


class LaunchFlops:
    """Context manager: counts the FLOPs of the kernels launched inside it."""

    def __enter__(self):
        torch = _lib.require_device()
        _lock.acquire()
        self._dev = torch.zeros(1, dtype=torch.int64, device="cuda")
        self.py = dict.fromkeys(KEYS, 0)
        self.counts: dict[str, int] = {}
        _lib.call("bt_flops_enable", self._dev.data_ptr())
        _active.cur = self
        return self

    def __exit__(self, *exc):
        torch = _lib.require_device()
        try:
            torch.cuda.synchronize()
            out = (C.c_longlong * 4)()
            _lib.call("bt_flops_read", C.cast(out, C.c_void_p))
        finally:
            _lib.call("bt_flops_enable", None)
            _active.cur = None
            _lock.release()
        self.counts = {k: int(out[i]) + self.py[k] for i, k in enumerate(KEYS)}
        self.counts["mha"] = int(self._dev.item())
        return False

    def add_to(self, counter) -> None:
        if counter is None:
            return
        for key in ("gemm0", "mha", "gemm1", "gemm2", "gemm3"):
            counter.add(key, self.counts[key])


def count_gemm(key: str, M: int, N: int, K: int) -> None:
    """A GEMM launched from Python adds its launch shape's FLOPs (no-op when
    no LaunchFlops is active)."""
    cur = getattr(_active, "cur", None)
    if cur is not None:
        cur.py[key] += 2 * int(M) * int(N) * int(K)
