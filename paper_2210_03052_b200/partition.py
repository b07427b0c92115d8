"""Token-balanced sequence partition across GPUs (north star: "Multi-GPU runs
split a variable-length batch across 1, 2, 4 and 8 GPUs ... by a
token-balanced partition with no collective on the hot path").

Sequences are independent units of the encoder (attention couples tokens only
within a sequence; every other op is per token, reference encoder.py:356-408),
so each rank runs ``forward`` on a contiguous range of sequences with no data
exchange.  Ranges are cut at quantiles of the prefix sum of per-sequence cost
c_i = 24 len_i k^2 + 4 len_i^2 k (one layer's FLOPs, flops.py:72-110), so the
slowest rank -- which sets the step time -- carries as little excess as a
contiguous cut allows.  Contiguous ranges keep the gathered output in the
original sequence order.

``gather_packed`` is the only collective: it assembles per-rank packed outputs
on every rank (NCCL all-gather over NVLink, gloo on CPU) when one result
tensor is required.  It is not on the timed hot path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


def sequence_cost(lengths, hidden: int) -> np.ndarray:
    n = np.asarray(lengths, dtype=np.float64)
    return 24.0 * n * hidden * hidden + 4.0 * n * n * hidden


@dataclass(frozen=True)
class Shard:
    rank: int
    start: int       # first sequence index (inclusive)
    stop: int        # last sequence index (exclusive)
    tokens: int
    cost: float

    @property
    def batch_size(self) -> int:
        return self.stop - self.start


def token_balanced_partition(lengths, world_size: int, hidden: int = 768) -> list[Shard]:
    """Contiguous ranges with (near-)equal cost.  Greedy boundary placement at
    the cost quantiles, then a local refinement that moves each boundary by one
    sequence while that lowers the maximum shard cost.  Every rank gets at
    least one sequence when there are enough sequences."""
    lens = [int(n) for n in lengths]
    n = len(lens)
    if world_size < 1:
        raise ValueError(f"world_size must be >= 1, got {world_size}")
    if n < world_size:
        raise ValueError(f"cannot split {n} sequences over {world_size} ranks")
    cost = sequence_cost(lens, hidden)
    pref = np.concatenate([[0.0], np.cumsum(cost)])
    total = pref[-1]
    bounds = [0]
    for r in range(1, world_size):
        target = total * r / world_size
        b = int(np.searchsorted(pref, target))
        # pick the closer of b-1 / b, keep strictly increasing and leave room
        if b > 0 and abs(pref[b - 1] - target) <= abs(pref[min(b, n)] - target):
            b -= 1
        b = max(b, bounds[-1] + 1)
        b = min(b, n - (world_size - r))
        bounds.append(b)
    bounds.append(n)

    def shard_costs(bd):
        return [pref[bd[i + 1]] - pref[bd[i]] for i in range(world_size)]

    improved = True
    while improved:
        improved = False
        for i in range(1, world_size):
            best = max(shard_costs(bounds))
            for delta in (-1, 1):
                nb = bounds[i] + delta
                if bounds[i - 1] < nb < bounds[i + 1]:
                    trial = bounds[:i] + [nb] + bounds[i + 1:]
                    if max(shard_costs(trial)) < best - 1e-9:
                        bounds, improved = trial, True
                        break
    return [Shard(r, bounds[r], bounds[r + 1], int(sum(lens[bounds[r]:bounds[r + 1]])),
                  float(pref[bounds[r + 1]] - pref[bounds[r]])) for r in range(world_size)]


def imbalance(shards: list[Shard]) -> float:
    """max shard cost / mean shard cost (1.0 = perfect)."""
    c = [s.cost for s in shards]
    return max(c) / (sum(c) / len(c))


def gather_packed(local_packed, shards: list[Shard], group=None):
    """All-gather variable-length packed outputs [T_r, k] into the global
    packed tensor [sum T_r, k] (rank order == sequence order).  Pads to the
    largest shard for the collective and trims."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    tmax = max(s.tokens for s in shards)
    k = local_packed.shape[1]
    buf = torch.zeros((tmax, k), dtype=local_packed.dtype, device=local_packed.device)
    buf[: local_packed.shape[0]] = local_packed
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([parts[s.rank][: s.tokens] for s in shards], dim=0)


def forward_sharded(weights, seqs, input_padded, config, *, group=None, gather: bool = True):
    """Multi-GPU encoder forward (reference
    ``forward``, encoder.py:411-437, split over ranks).

    Every rank holds the whole batch description and input; it runs the
    padding-free GPU engine on its contiguous token-balanced shard of
    sequences only (no collective on the hot path).  With ``gather`` the
    valid output rows of every shard are all-gathered (``gather_packed``:
    NCCL over NVLink, or gloo through host memory) and unpacked on the device
    into the one padded ``[bs*mx, k]`` result the reference returns, on every
    rank.  Without ``gather`` the rank's own padded shard output is returned.

    Output type follows the input, as ``forward``: a CUDA tensor for a CUDA
    input, a host ``Tensor`` otherwise.  Per-sequence results do not depend
    on the partition when the forward runs the one-problem-per-tile MHA
    (max_seq_len > 256 or batch > 256; the segment kernel that groups short
    sequences for small batches shifts their keys inside a block, which
    changes bf16 rounding only) and the shard and the full batch make the
    same GEMM + LayerNorm fusion choice (the fused kernel runs when a batch's
    128-row blocks fit one wave of clusters, ``bt_fused_attn_out_ln`` /
    ``bt_fused_ffn2_ln``; it rounds the projection differently, within
    tolerance): tests/test_gpu_determinism.py."""
    from dataclasses import replace

    import torch
    import torch.distributed as dist

    from .encoder import as_model_config, forward
    from .packing import as_seq_lengths, pack_device, plan_for_lengths, unpack_device
    from .tensor import Tensor, host_array, is_device

    config = as_model_config(config)
    seqs = as_seq_lengths(seqs)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    shards = token_balanced_partition(seqs.lengths, world, config.hidden_dim)
    sh = shards[rank]
    mx = seqs.max_seq_len
    local_seqs = type(seqs).of(list(seqs.lengths[sh.start:sh.stop]), mx)
    local_cfg = replace(config, batch_size=sh.batch_size)
    device_io = is_device(input_padded)
    if device_io:
        x_local = input_padded[sh.start * mx: sh.stop * mx].to(torch.float32).contiguous()
    else:
        x_local = torch.from_numpy(np.ascontiguousarray(host_array(input_padded)[sh.start * mx: sh.stop * mx])).to(
            "cuda")
    y_local = forward(weights, local_seqs, x_local, local_cfg)  # CUDA fp32 [n_r*mx, k]
    if not gather or world == 1:
        return y_local if device_io else Tensor(y_local.cpu().numpy())
    packed_local = pack_device(y_local, plan_for_lengths(local_seqs))  # [T_r, k] fp32
    on_host = dist.get_backend(group) != "nccl"
    g = gather_packed(packed_local.cpu() if on_host else packed_local, shards, group)
    full = unpack_device(g.to("cuda"), plan_for_lengths(seqs))
    return full if device_io else Tensor(full.cpu().numpy())
