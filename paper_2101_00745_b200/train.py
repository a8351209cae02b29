"""Synthetic-data training throughput of the SCC models (images/sec), one
process per GPU, data parallel over NCCL.

Every world size runs the same step: forward, cross-entropy, backward, ONE
bucketed all-reduce (mean) of all gradients through ``dist.GradSync`` (a
no-op at world size 1), momentum SGD update -- captured once as a CUDA graph
and replayed, collective included.  ``tests/test_dist.py`` runs this same
``make_train_step`` / ``GradSync`` code with 2 gloo ranks on CPU.

The reference trains its sequential networks on one CPU thread pool
(train.cpp:66-125); this is the B200 harness for BASELINE configs C2-C4
(SCC-VGG16 / SCC-ResNet-18 on CIFAR-shaped and SCC-ResNet-50 on
ImageNet-shaped synthetic data).
"""
from __future__ import annotations

import torch
import torch.distributed as dist
from torch import nn

from .dist import GradSync
from .models import MODELS


def make_train_step(model: nn.Module, opt: torch.optim.Optimizer, loss_fn, x: torch.Tensor,
                    y: torch.Tensor, sync: GradSync):
    """One data-parallel SGD step over this rank's shard (x, y)."""

    def step():
        opt.zero_grad(set_to_none=False)
        loss = loss_fn(model(x), y)
        loss.backward()
        sync()
        opt.step()
        return loss

    return step


def train_throughput(model_name: str = "resnet18", batch: int = 128, steps: int = 20, warmup: int = 5,
                     image: int = 32, num_classes: int = 10, seed: int = 0, graph: bool = True):
    """Time `steps` SGD steps after `warmup` steps.  Returns images/sec over
    all ranks (per-rank batch x world size / max-over-ranks device time).

    The whole step is captured once as a CUDA graph and replayed (a
    CIFAR-size step is ~300 small kernels, so eager launches make it host
    bound); the warm-up runs on the capture stream so every per-stream
    resource of the SCC plans (and NCCL's) exists before capture."""
    dev = torch.device("cuda", torch.cuda.current_device())
    ws = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    # fp32 end to end: the stock dense layers (stem, 1x1 convs, head) must not
    # silently run TF32 next to the 3xTF32 SCC kernels
    tf32 = (torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32)
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        return _train_throughput(model_name, batch, steps, warmup, image, num_classes, seed, graph, dev, ws)
    finally:
        torch.backends.cudnn.allow_tf32, torch.backends.cuda.matmul.allow_tf32 = tf32


def _train_throughput(model_name, batch, steps, warmup, image, num_classes, seed, graph, dev, ws):
    torch.manual_seed(seed)
    model = MODELS[model_name](num_classes=num_classes, device=dev)
    sync = GradSync(model)
    sync.broadcast_parameters()
    opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9, weight_decay=5e-4)
    gen = torch.Generator(device=dev).manual_seed(seed + (dist.get_rank() if ws > 1 else 0))
    x = torch.randn(batch, 3, image, image, device=dev, generator=gen)
    y = torch.randint(0, num_classes, (batch,), device=dev, generator=gen)
    step = make_train_step(model, opt, nn.CrossEntropyLoss(), x, y, sync)

    launch = "eager"
    stream = torch.cuda.Stream(dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(stream):
        losses = [float(step().item()) for _ in range(max(warmup, 1))]
        run = step
        if graph:
            try:
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    static_loss = step()
                g.replay()
                stream.synchronize()

                def run():
                    g.replay()
                    return static_loss

                launch = "cuda-graph"
            except Exception:  # capture unsupported here: keep eager launches
                run = step
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            last = run()
        e1.record(stream)
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    return {"model": f"SCC-{model_name}", "images_per_s": round(batch * ws / (ms * 1e-3), 1),
            "ms_per_step": round(ms, 4), "batch_per_gpu": batch, "global_batch": batch * ws,
            "n_gpus": ws, "steps": steps, "warmup": warmup, "image": f"3x{image}x{image}",
            "loss_first": round(losses[0], 4), "loss_last": round(float(last.item()), 4),
            "launch": launch, "dense_layers": "fp32 (TF32 off)",
            "data": "synthetic N(0,1) images, uniform labels"}
