"""Optimisation-ladder variants (reference bench.py:35-41, encoder.py:367-408)
on the B200: every OptFlags subset other than all_on()."""

from __future__ import annotations

from .errors import ConfigError


def forward_variant(weights, seqs, input_padded, config, *, counter=None):
    raise ConfigError(f"OptFlags {config.flags} is not implemented on the B200 path yet; use OptFlags.all_on()")


def encoder_layer_variant(x, layer, config, plan, *, counter=None):
    raise ConfigError(f"OptFlags {config.flags} is not implemented on the B200 path yet; use OptFlags.all_on()")
