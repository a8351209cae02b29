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
        # single flat bucket, reduced in place (bench.py's dW|db buffer)
        g3 = torch.full((4,), float(rank + 1))
        allreduce_grads([g3], average=False)
        ok = ok and torch.equal(g3, torch.full((4,), 3.0))
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


# --- the data-parallel training step the GPU harness runs (train.py) --------


def _tiny_model():
    torch.manual_seed(3)
    return torch.nn.Sequential(torch.nn.Conv2d(3, 4, 3, padding=1), torch.nn.ReLU(), torch.nn.Flatten(),
                               torch.nn.Linear(4 * 6 * 6, 5))


def _train_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2101_00745_b200.dist import GradSync, shard_batch
        from paper_2101_00745_b200.train import make_train_step
        model = _tiny_model()
        if rank == 1:  # diverged start: broadcast_parameters must fix it
            with torch.no_grad():
                for p in model.parameters():
                    p.add_(1.0)
        sync = GradSync(model)
        sync.broadcast_parameters()
        g = torch.Generator().manual_seed(11)
        x = torch.randn(8, 3, 6, 6, generator=g)
        y = torch.randint(0, 5, (8,), generator=g)
        opt = torch.optim.SGD(model.parameters(), lr=0.1, momentum=0.9)
        step = make_train_step(model, opt, torch.nn.CrossEntropyLoss(), shard_batch(x, rank, world),
                               shard_batch(y, rank, world), sync)
        for _ in range(3):
            step()
        # single-process full-batch reference of the same 3 steps
        ref = _tiny_model()
        ropt = torch.optim.SGD(ref.parameters(), lr=0.1, momentum=0.9)
        rstep = make_train_step(ref, ropt, torch.nn.CrossEntropyLoss(), x, y, lambda: None)
        for _ in range(3):
            rstep()
        ok = all(torch.allclose(a, b, rtol=1e-5, atol=1e-6) for a, b in zip(model.parameters(), ref.parameters()))
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_two_rank_gloo_train_step_matches_full_batch():
    """train.make_train_step + dist.GradSync (what train_throughput runs, and
    captures in a CUDA graph on GPUs) on 2 gloo ranks == one full-batch step."""
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0, 0])
    port = _free_port()
    procs = [ctx.Process(target=_train_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=180)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    assert list(out) == [1, 1]


def test_scc_parameters_cover_dsc_blocks():
    """SccGradSync must see both halves of every DSC2d block."""
    from paper_2101_00745_b200.dist import SccGradSync, scc_parameters
    from paper_2101_00745_b200.models import SCCResNet18
    m = SCCResNet18()
    names = {id(p) for p in scc_parameters(m)}
    want = set()
    for mod in m.modules():
        if type(mod).__name__ == "DSC":
            want |= {id(mod.dw_weight), id(mod.weight)}
    assert want and want <= names
    assert len(SccGradSync(m).params) == len(names)


def test_flat_allreduce_in_place_single_rank():
    """bench.py's flat dW|db bucket path: world size 1 is a no-op."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dist.init_process_group("gloo", rank=0, world_size=1)
    try:
        t = torch.arange(6, dtype=torch.float32)
        allreduce_grads([t])
        assert torch.equal(t, torch.arange(6, dtype=torch.float32))
    finally:
        dist.destroy_process_group()
