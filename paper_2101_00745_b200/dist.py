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


def _world(group=None) -> int:
    """World size, 1 when no process group is initialised (single process)."""
    if not (dist.is_available() and dist.is_initialized()):
        return 1
    return dist.get_world_size(group)


def allreduce_grads(grads: List[torch.Tensor], group=None, average: bool = True,
                    bucket: Optional[GradBucket] = None) -> None:
    """Sum (or mean) `grads` across the process group in ONE collective.  A
    single contiguous tensor (an already-flat bucket, as bench.py's dW|db
    buffer) is reduced in place with no pack / unpack copies."""
    if not grads:
        return
    world = _world(group)
    if world == 1:
        return
    if len(grads) == 1 and grads[0].is_contiguous():
        flat = grads[0]
        dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
        if average:
            flat.div_(world)
        return
    bucket = bucket or GradBucket(grads)
    flat = bucket.pack(grads)
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    if average:
        flat.div_(world)
    bucket.unpack(grads)


def scc_parameters(module: torch.nn.Module) -> Iterable[torch.nn.Parameter]:
    """The parameters of every SCC stage: SCC2d layers and both halves of the
    DSC2d (depthwise 3x3 + SCC) blocks the model zoo is built from."""
    from .module import DSC2d, SCC2d
    for m in module.modules():
        if isinstance(m, (SCC2d, DSC2d)):
            for name in ("dw_weight", "dw_bias", "weight", "bias"):
                p = getattr(m, name, None)
                if p is not None:
                    yield p


class GradSync:
    """Data-parallel gradient exchange of a whole model: after
    loss.backward(), ONE bucketed all-reduce (mean) of every parameter
    gradient.  All tensors live in fixed buffers, so the call can be captured
    in the same CUDA graph as the step (NCCL collectives are graph-capturable)
    and the N-GPU step replays exactly like the 1-GPU one.  World size 1 is a
    no-op.  `params` defaults to every trainable parameter of `module`."""

    def __init__(self, module: torch.nn.Module, group=None, average: bool = True,
                 params: Optional[Sequence[torch.nn.Parameter]] = None):
        self.params = [p for p in (params if params is not None else module.parameters())
                       if p.requires_grad]
        self.group, self.average = group, average
        self._bucket = GradBucket(self.params) if self.params else None

    def broadcast_parameters(self, src: int = 0) -> None:
        """Start every rank from rank `src`'s weights (one collective)."""
        if not self.params or _world(self.group) == 1:
            return
        flat = self._bucket.pack([p.detach() for p in self.params])
        dist.broadcast(flat, src=src, group=self.group)
        with torch.no_grad():
            self._bucket.unpack([p.data for p in self.params])

    def __call__(self) -> None:
        if not self.params or _world(self.group) == 1:
            return
        grads = []
        for p in self.params:
            if p.grad is None:  # a parameter this step did not reach: zero, so every rank reduces alike
                p.grad = torch.zeros_like(p)
            grads.append(p.grad)
        allreduce_grads(grads, self.group, self.average, self._bucket)


class SccGradSync(GradSync):
    """GradSync over the SCC stages only (SCC2d, and DSC2d's depthwise + SCC
    parameters), for callers that leave the other parameters to DDP."""

    def __init__(self, module: torch.nn.Module, group=None, average: bool = True):
        super().__init__(module, group, average, params=list(scc_parameters(module)))
