"""Multi-process coverage of the token-balanced partition (north star:
"split a variable-length batch across 1, 2, 4 and 8 GPUs ... with no
collective on the hot path; NCCL only to gather outputs where a single
result tensor is required").

Runs here on CPU: world_size-2 torch.distributed with the gloo backend.  Each
rank takes its shard of the batch from token_balanced_partition, runs the CPU
oracle forward on it (the GPU path is exercised by the -m gpu tests; this
test covers the sharding and gather logic), and gather_packed assembles the
packed outputs; every rank must hold the single-process result."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import packbert_np as orc


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, result_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_03052_b200.harness import gen_lengths
        from paper_2210_03052_b200.partition import gather_packed, token_balanced_partition

        bs, mx, hid = 9, 48, 128
        lens = list(gen_lengths(bs, mx, "fixed", seed=3, alpha=0.6).lengths)
        shards = token_balanced_partition(lens, world, hid)
        mine = shards[rank]
        cfg = orc.OracleConfig(1, 2, 64, mx, mine.batch_size)
        w = orc.stress_weights(orc.OracleConfig(1, 2, 64, mx, bs), 0)
        x_all = orc.gen_input(lens, mx, hid, 0)
        x_local = x_all[mine.start * mx: mine.stop * mx]
        local_lens = lens[mine.start:mine.stop]
        y_local = orc.forward(w, local_lens, x_local, cfg)
        offs, _, _ = orc.compute_plan(orc.build_mask(local_lens, mx))
        packed_local = torch.from_numpy(y_local[offs])
        gathered = gather_packed(packed_local, shards).numpy()
        result_q.put((rank, gathered, [(s.start, s.stop, s.tokens) for s in shards]))
    finally:
        dist.destroy_process_group()


def test_partition_and_gather_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_2210_03052_b200.harness import gen_lengths

    bs, mx, hid = 9, 48, 128
    lens = list(gen_lengths(bs, mx, "fixed", seed=3, alpha=0.6).lengths)
    full = orc.forward(orc.stress_weights(orc.OracleConfig(1, 2, 64, mx, bs), 0), lens, orc.gen_input(lens, mx, hid, 0),
                       orc.OracleConfig(1, 2, 64, mx, bs))
    offs, _, _ = orc.compute_plan(orc.build_mask(lens, mx))
    want = full[offs]
    shard_sets = {tuple(r[2]) for r in results}
    assert len(shard_sets) == 1, "ranks disagree on the partition"
    (start0, stop0, _), (start1, stop1, _) = results[0][2]
    assert start0 == 0 and stop0 == start1 and stop1 == bs
    for rank, gathered, _ in results:
        assert gathered.shape == want.shape
        # per-sequence work is independent of batch composition up to BLAS blocking
        np.testing.assert_allclose(gathered, want, rtol=1e-4, atol=1e-5)
