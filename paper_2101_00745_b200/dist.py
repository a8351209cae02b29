"""Data-parallel plumbing for SCC layers (north_star: batches shard across the
GPUs of one box; the SCC weight gradients are all-reduced over NVLink).

The operator shards naturally by batch: forward and
backward-data are independent per sample, backward-weight reduces over
(n, p), so each rank computes partial dW/db on its samples and one all-reduce
(sum, then 1/world for a mean) completes the step.  The gradients are tiny
(c_out*gw + c_out floats per layer), so every SCC gradient of a model goes in
ONE flat bucket and one collective per step: latency-bound traffic is batched,
not split per layer.  Backend: NCCL on GPUs, gloo for CPU tests.
"""
from __future__ import annotations

from typing import Iterable, List, Optional, Sequence

import torch
import torch.distributed as dist


def shard_range(count: int, rank: int, world: int):
    """Contiguous [begin, end) of `count` items for `rank` -- the same
    partition rule as the reference's parallel_chunks (parallel.cpp:56-61)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} / world {world}")
    return count * rank // world, count * (rank + 1) // world


def shard_batch(t: torch.Tensor, rank: int, world: int) -> torch.Tensor:
    b, e = shard_range(t.shape[0], rank, world)
    return t[b:e]


class GradBucket:
    """One flat buffer holding the gradients of a fixed list of tensors."""

    def __init__(self, params: Sequence[torch.Tensor]):
        self.params = list(params)
        numel = sum(p.numel() for p in self.params)
        dev = self.params[0].device if self.params else torch.device("cpu")
        dtype = self.params[0].dtype if self.params else torch.float32
        self.flat = torch.zeros(numel, dtype=dtype, device=dev)

    def pack(self, grads: Sequence[torch.Tensor]) -> torch.Tensor:
        off = 0
        for g in grads:
            n = g.numel()
            self.flat[off:off + n].copy_(g.reshape(-1))
            off += n
        return self.flat

    def unpack(self, grads: Sequence[torch.Tensor]) -> None:
        off = 0
        for g in grads:
            n = g.numel()
            g.copy_(self.flat[off:off + n].view_as(g))
            off += n


def allreduce_grads(grads: List[torch.Tensor], group=None, average: bool = True,
                    bucket: Optional[GradBucket] = None) -> None:
    """Sum (or mean) `grads` across the process group in ONE collective."""
    if not grads:
        return
    world = dist.get_world_size(group)
    if world == 1:
        return
    bucket = bucket or GradBucket(grads)
    flat = bucket.pack(grads)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if average:
        flat.div_(world)
    bucket.unpack(grads)


def scc_parameters(module: torch.nn.Module) -> Iterable[torch.nn.Parameter]:
    from .module import SCC2d
    for m in module.modules():
        if isinstance(m, SCC2d):
            yield m.weight
            if m.bias is not None:
                yield m.bias


class SccGradSync:
    """Call after loss.backward(): one bucketed all-reduce of every SCC
    parameter gradient of `module` (other parameters are left to the caller's
    DDP wrapper)."""

    def __init__(self, module: torch.nn.Module, group=None, average: bool = True):
        self.params = [p for p in scc_parameters(module) if p.requires_grad]
        self.group, self.average = group, average
        self._bucket = None

    def __call__(self) -> None:
        grads = [p.grad for p in self.params if p.grad is not None]
        if not grads:
            return
        if self._bucket is None or len(self._bucket.params) != len(grads):
            self._bucket = GradBucket(grads)
        allreduce_grads(grads, self.group, self.average, self._bucket)
