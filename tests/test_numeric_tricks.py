"""Host (numpy, fp32) emulation of the device-side numeric tricks, so their
accuracy claims are checked without a GPU: the FMA-pipe exp2 of the MHA
softmax (ptx.cuh ex2_poly2) must stay below bf16's 2^-9 relative step and
return exactly 0 for masked (-inf) keys."""

import numpy as np


def _ex2_poly(x):
    x = np.asarray(x, np.float32)
    xc = np.maximum(x, np.float32(-127))
    magic = np.float32(12582912.0)
    t = (xc + magic).astype(np.float32)
    fr = (xc - (t - magic)).astype(np.float32)
    p = np.float32(0.05484628) * fr + np.float32(0.24180230)
    p = (p * fr + np.float32(0.69324806)).astype(np.float32)
    p = (p * fr + np.float32(0.99998888)).astype(np.float32)
    scale = ((t.view(np.int32) - np.int32(0x4B400000 - 127)) << 23).astype(np.int32).view(np.float32)
    return (p * scale).astype(np.float32)


def test_ex2_poly_accuracy():
    x = np.linspace(-126, 8.5, 400001, dtype=np.float32)  # softmax exponents: <= 8 (lazy max threshold)
    y = _ex2_poly(x)
    ref = np.exp2(x.astype(np.float64))
    assert (np.abs(y - ref) / ref).max() < 2.5e-4 < 2.0 ** -9


def test_ex2_poly_masked_is_zero():
    y = _ex2_poly(np.array([-np.inf, -1e30, -200.0, -127.0, -126.6], np.float32))
    assert np.all(y == 0.0) and not np.signbit(y).any()
