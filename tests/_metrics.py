"""Numerical comparison helpers shared by the parity tests."""

import numpy as np


def as_np(x):
    if hasattr(x, "array"):
        x = x.array
    if hasattr(x, "detach"):
        x = x.detach().float().cpu().numpy()
    return np.asarray(x, dtype=np.float64)


def rel_fro(a, b):
    a, b = as_np(a), as_np(b)
    d = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (d if d else 1.0))


def cosine(a, b):
    a, b = as_np(a).ravel(), as_np(b).ravel()
    na, nb = np.linalg.norm(a), np.linalg.norm(b)
    if na == 0 and nb == 0:
        return 1.0
    return float(a @ b / (na * nb))


def max_abs(a, b):
    return float(np.max(np.abs(as_np(a) - as_np(b)))) if as_np(a).size else 0.0


def rms(a):
    a = as_np(a)
    return float(np.sqrt(np.mean(a * a))) if a.size else 0.0


def assert_close_bf16(got, want, *, cos_min=0.9999, rel_max=1.5e-2, max_abs_max=None, what=""):
    """north-star tolerance (BASELINE.json): cosine >= 0.9999 and a bounded
    max-abs error; relFro bound per SURVEY.md section 8(c)."""
    c, r, m = cosine(got, want), rel_fro(got, want), max_abs(got, want)
    msg = f"{what}: cosine={c:.6f} relFro={r:.3e} maxabs={m:.3e}"
    assert c >= cos_min, msg
    assert r <= rel_max, msg
    if max_abs_max is not None:
        assert m <= max_abs_max, msg
    return c, r, m
