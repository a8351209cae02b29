"""Multi-process (world_size 2, gloo, CPU) test of the data-parallel path:
batch sharding + one bucketed all-reduce of the SCC gradients reproduces the
full-batch gradients.  Per-rank gradients come from the CPU
oracle, so this runs without a GPU; the GPU run of the same path is
`torchrun ... bench.py --gpus N` (NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2101_00745_b200.dist import GradBucket, allreduce_grads, shard_range


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import load_port
        port_o = load_port()
        cfg = port_o.config(24, 40, 3, ("channels", 2), True)
        rng = np.random.default_rng(9)
        n = 7  # uneven split on purpose
        x = rng.standard_normal((n, 24, 5, 5))
        dy = rng.standard_normal((n, 40, 5, 5))
        b, e = shard_range(n, rank, world)
        dw, db = port_o.backward_params(cfg, dy[b:e], x[b:e])
        g_w = torch.from_numpy(dw.copy())
        g_b = torch.from_numpy(db.copy())
        allreduce_grads([g_w, g_b], average=False)
        full_w, full_b = port_o.backward_params(cfg, dy, x)
        ok = (np.allclose(g_w.numpy(), full_w, rtol=0, atol=1e-12 * np.abs(full_w).max())
              and np.allclose(g_b.numpy(), full_b, rtol=0, atol=1e-12 * np.abs(full_b).max()))
        # mean variant
        g2 = [torch.full((3,), float(rank + 1), dtype=torch.float64)]
        allreduce_grads(g2, average=True)
        ok = ok and torch.allclose(g2[0], torch.full((3,), 1.5, dtype=torch.float64))
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_shard_range_partition():
    for n in (0, 1, 7, 32, 33):
        for world in (1, 2, 3, 8):
            spans = [shard_range(n, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(spans[i][1] == spans[i + 1][0] for i in range(world - 1))


def test_bucket_roundtrip():
    a, b = torch.randn(3, 4), torch.randn(5)
    bk = GradBucket([a, b])
    flat = bk.pack([a, b]).clone()
    a2, b2 = torch.zeros_like(a), torch.zeros_like(b)
    bk.flat.copy_(flat)
    bk.unpack([a2, b2])
    assert torch.equal(a, a2) and torch.equal(b, b2)


def test_two_rank_gloo_allreduce_matches_full_batch():
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0, 0])
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=120)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert list(out) == [1, 1]
