"""The optimisation ladder on the B200 (reference bench.py:35-41 LADDER and
the OptFlags branches of encoder.py:367-408; paper Fig. 9 / Table III).

Every OptFlags subset runs on the same sm_100a kernels:

  baseline          padded layout [bs*mx, k]: GEMMs over every padded row,
                    padded MHA (mx x mx rectangle, -1e9-equivalent key mask,
                    padded query rows zeroed), LN as three passes
                    (add, add bias, layernorm), FFN bias + GELU as a separate pass
  layernorm_fusion  + one-pass add-bias+residual+LN
  bias_gelu_fusion  + bias + GELU in the FFN1 GEMM epilogue
  rm_padding        + packed [T, k] everywhere except attention, which is
                    bracketed by unpack / pack around the padded MHA
  fused_mha         + varlen MHA straight on the packed layout (= all_on())

Activations are bf16 between kernels in every rung, so rungs differ only in
which work is done, not in precision.  Each rung is checked against the
reference's own outputs (tests/golden/encoder.npz tiny_padded / tiny_rmpad)
and against one another.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ShapeError
from .packing import PackingPlan, ensure_plan, pack_device, plan_for_lengths, unpack_device
from .tensor import FlopCounter, Tensor, host_array, is_device

LADDER_NAMES = ["baseline", "layernorm_fusion", "bias_gelu_fusion", "rm_padding", "fused_mha"]


def ladder_flags(name: str):
    from .encoder import OptFlags

    table = {
        "baseline": OptFlags(),
        "layernorm_fusion": OptFlags(fuse_layernorm=True),
        "bias_gelu_fusion": OptFlags(fuse_layernorm=True, fuse_bias_gelu=True),
        "rm_padding": OptFlags(fuse_layernorm=True, fuse_bias_gelu=True, zero_padding=True),
        "fused_mha": OptFlags.all_on(),
    }
    return table[name]


def mha_padded_device(qkv_bf16, plan: PackingPlan, head_num: int, head_size: int, out=None):
    """mha_baseline (attention.py:135-174) on a padded [bs*mx, 3k] QKV tensor."""
    torch = _lib.require_device()
    rows = plan.padded_rows
    hidden = head_num * head_size
    if tuple(qkv_bf16.shape) != (rows, 3 * hidden):
        raise ShapeError(f"padded qkv must be [{rows}, {3 * hidden}], got {tuple(qkv_bf16.shape)}")
    if out is None:
        out = torch.empty((rows, hidden), dtype=torch.bfloat16, device=qkv_bf16.device)
    _lib.call("bt_mha_padded", qkv_bf16.data_ptr(), plan.seq_starts_dev.data_ptr(), plan.batch_size,
              plan.max_seq_len, head_num, head_size, out.data_ptr(), _lib.stream_ptr())
    return out


def _ln_unfused(a, residual, bias, gamma, beta, eps):
    """layernorm(add_rowvec(add(a, residual), bias)) as three device passes
    (encoder.py:390, 408): add, add bias, LN."""
    from .fusion import add_device, bias_act_device, ln_device

    t = add_device(a, residual)
    t = bias_act_device(t, bias, 0)
    return ln_device(t, None, None, gamma, beta, eps)


def layer_variant_device(dl, x, plan: PackingPlan, config, flags):
    """One encoder layer on device bf16 activations for any OptFlags subset;
    `dl` is a DeviceLayer (uploaded weights), x is packed iff zero_padding."""
    from .attention import mha_device
    from .fusion import bias_act_device, ln_device
    from .tensor import gemm_device

    from .instrument import count_gemm

    k = config.hidden_dim
    f = config.ffn_scale * k
    m = int(x.shape[0])
    qkv = gemm_device(x, dl.qkv_w, dl.qkv_b, None, _lib.EPI_BIAS)  # Q/K/V biases (added on load in the reference)
    count_gemm("gemm0", m, 3 * k, k)
    if not flags.zero_padding:
        attn = mha_padded_device(qkv, plan, config.head_num, config.head_size)
    elif not flags.fused_mha:
        qkv_p = unpack_device(qkv, plan, out_dtype=qkv.dtype)
        attn = pack_device(mha_padded_device(qkv_p, plan, config.head_num, config.head_size), plan)
    else:
        attn = mha_device(qkv, plan, config.head_num, config.head_size, cutoff=config.cutoff,
                          split_seq_len=config.split_seq_len)
    proj = gemm_device(attn, dl.ao_w)
    count_gemm("gemm1", m, k, k)
    if flags.fuse_layernorm:
        y0 = ln_device(proj, x, dl.ao_b, dl.ln0_g, dl.ln0_b, dl.ln0_eps)
    else:
        y0 = _ln_unfused(proj, x, dl.ao_b, dl.ln0_g, dl.ln0_b, dl.ln0_eps)
    if flags.fuse_bias_gelu:
        h1 = gemm_device(y0, dl.w1, dl.b1, None, _lib.EPI_BIAS_GELU)
    else:
        h1 = bias_act_device(gemm_device(y0, dl.w1), dl.b1, 1)
    count_gemm("gemm2", m, f, k)
    h2 = gemm_device(h1, dl.w2)
    count_gemm("gemm3", m, k, f)
    if flags.fuse_layernorm:
        return ln_device(h2, y0, dl.b2, dl.ln1_g, dl.ln1_b, dl.ln1_eps)
    return _ln_unfused(h2, y0, dl.b2, dl.ln1_g, dl.ln1_b, dl.ln1_eps)


def forward_variant_device(eng, plan: PackingPlan, x_padded_f32, config):
    """Device forward for any OptFlags subset: fp32 padded in, fp32 out
    (padded layout; padded rows exactly zero iff zero_padding)."""
    torch = _lib.require_device()
    flags = config.flags
    if flags.zero_padding:
        x = pack_device(x_padded_f32, plan, out_dtype=torch.bfloat16)
    else:
        x = x_padded_f32.to(torch.bfloat16)
    for li in range(config.layers):
        x = layer_variant_device(eng.layer(li), x, plan, config, flags)
    if flags.zero_padding:
        return unpack_device(x, plan)
    return x.float()


def forward_variant(weights, seqs, input_padded, config, *, counter=None):
    """forward() for OptFlags other than all_on() (reference encoder.py:411-437)."""
    from .encoder import engine_for

    torch = _lib.require_device()
    eng = engine_for(weights, config)
    plan = plan_for_lengths(seqs)
    device_mode = is_device(input_padded)
    x = input_padded.to(torch.float32).contiguous() if device_mode else torch.from_numpy(
        host_array(input_padded)).to("cuda")
    if counter is None:
        out = forward_variant_device(eng, plan, x, config)
    else:
        from .instrument import LaunchFlops

        with LaunchFlops() as lf:
            out = forward_variant_device(eng, plan, x, config)
        lf.add_to(counter)
    return out if device_mode else Tensor(out.cpu().numpy())


def encoder_layer_variant(x, layer, config, plan, *, counter=None):
    """encoder_layer() for OptFlags other than all_on() (encoder.py:337-408)."""
    from .encoder import engine_for_layer

    torch = _lib.require_device()
    plan = ensure_plan(plan)
    eng = engine_for_layer(layer, config)
    device_mode = is_device(x)
    xb = x.to(torch.bfloat16).contiguous() if device_mode else torch.from_numpy(host_array(x)).to("cuda").to(
        torch.bfloat16)
    if counter is None:
        y = layer_variant_device(eng.layer(0), xb, plan, config, config.flags)
    else:
        from .instrument import LaunchFlops

        with LaunchFlops() as lf:
            y = layer_variant_device(eng.layer(0), xb, plan, config, config.flags)
        lf.add_to(counter)
    return y.float() if device_mode else Tensor(y.float().cpu().numpy())
