"""Benchmark-harness pieces the reference ships (bench.py, flops.py) restated
for the B200 package: the seeded synthetic-input generators, the exact FLOP
model, and the algorithmic byte model used for the roofline fractions.

The generators reproduce the reference's draws exactly (checked against the
reference's frozen outputs in tests/test_host_api.py), so the GPU path, the
CPU oracle and the reference all see identical data.
"""

from __future__ import annotations

import numpy as np

from .errors import ConfigError
from .packing import SeqLengths, build_mask


def gen_lengths(batch_size: int, max_seq_len: int, mode: str = "uniform", seed: int = 0,
                alpha: float | None = None) -> SeqLengths:
    """Uniform integer lengths in [1, max]; "fixed" then nudges entries
    round-robin (clamped to [1, max]) until the total is round(alpha * max *
    batch) (reference bench.py:58-98)."""
    if mode not in ("uniform", "fixed"):
        raise ConfigError(f"unknown length mode {mode!r}; choose 'uniform' or 'fixed'")
    rng = np.random.default_rng(seed)
    lengths = rng.integers(1, max_seq_len + 1, size=batch_size).astype(np.int64)
    if mode == "fixed":
        if alpha is None:
            raise ConfigError("fixed mode requires alpha")
        if not 0.0 < alpha <= 1.0:
            raise ConfigError(f"alpha must be in (0, 1], got {alpha}")
        if alpha * max_seq_len < 1.0:
            raise ConfigError(f"alpha * max_seq_len = {alpha * max_seq_len:.3f} < 1: no valid lengths exist")
        target = int(round(alpha * max_seq_len * batch_size))
        target = min(max(target, batch_size), batch_size * max_seq_len)
        remaining = target - int(lengths.sum())
        cursor = 0
        while remaining != 0:
            j = cursor % batch_size
            if remaining > 0 and lengths[j] < max_seq_len:
                lengths[j] += 1
                remaining -= 1
            elif remaining < 0 and lengths[j] > 1:
                lengths[j] -= 1
                remaining += 1
            cursor += 1
    return SeqLengths.of(lengths.tolist(), max_seq_len)


def gen_input(seqs: SeqLengths, hidden: int, seed: int) -> np.ndarray:
    """N(0,1) fp32 padded input from default_rng(seed + 1), padded rows zero
    (reference bench.py:181-186)."""
    rng = np.random.default_rng(seed + 1)
    data = rng.standard_normal((seqs.batch_size * seqs.max_seq_len, hidden)).astype(np.float32)
    data[~build_mask(seqs).reshape(-1).astype(bool)] = 0.0
    return data


def layer_flops(lengths, hidden: int, ffn_scale: int = 4) -> dict[str, int]:
    """Exact per-layer FLOPs of the padding-free fused variant (reference
    flops.py:72-110, variant zero_padding_fused_mha)."""
    T = int(sum(lengths))
    k = hidden
    f = 2 * ffn_scale
    return {"gemm0": 6 * T * k * k, "mha": 4 * int(sum(int(n) * int(n) for n in lengths)) * k,
            "gemm1": 2 * T * k * k, "gemm2": f * T * k * k, "gemm3": f * T * k * k}


def forward_flops(lengths, hidden: int, layers: int, ffn_scale: int = 4) -> int:
    return layers * sum(layer_flops(lengths, hidden, ffn_scale).values())


def kernel_bytes(kind: str, T: int, k: int, bs: int = 0, mx: int = 0) -> int:
    """Algorithmic HBM bytes per launch of the memory-bound kernels
    (SURVEY.md section 8d): bf16 activations, fp32 padded I/O."""
    if kind == "ln":        # read x, read residual, write y (bf16)
        return 3 * T * k * 2
    if kind == "pack":      # fp32 valid rows in, bf16 packed out, int32 seq_starts
        return T * k * 4 + T * k * 2 + 4 * (bs + 1)
    if kind == "unpack":    # bf16 packed in, fp32 padded out (zeros included)
        return T * k * 2 + bs * mx * k * 4
    if kind == "plan":      # int32 lengths in, seq_starts + (start, length) schedule out
        return 4 * bs + 4 * (bs + 1) + 8 * bs
    if kind == "prologue":  # plan + pack + the zeroed padded output rows (fp32) + row_map
        return (4 * bs + 4 * (bs + 1) + 8 * bs) + (T * k * 4 + T * k * 2) + (bs * mx - T) * k * 4 + 4 * T
    if kind == "ln_out":    # read x, read residual (bf16), write the fp32 output rows
        return 2 * T * k * 2 + T * k * 4
    raise ValueError(kind)
