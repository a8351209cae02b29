"""Synthetic-data training throughput of the SCC models (images/sec), one
process per GPU, data parallel over NCCL (DistributedDataParallel: one
bucketed all-reduce of the gradients, SCC weights included, per step).

The reference trains its sequential networks on one CPU thread pool
(train.cpp:66-125); this is the B200 harness for BASELINE configs C2/C3
(SCC-VGG16 / SCC-ResNet-18 on CIFAR-shaped synthetic data).
"""
from __future__ import annotations

import torch
import torch.distributed as dist
from torch import nn

from .models import MODELS


def train_throughput(model_name: str = "resnet18", batch: int = 128, steps: int = 20, warmup: int = 5,
                     image: int = 32, num_classes: int = 10, seed: int = 0, graph: bool = True):
    """Time `steps` SGD steps (forward, cross-entropy, backward, all-reduce
    when distributed, momentum SGD update) after `warmup` steps.  Returns
    per-rank images/sec x world size (max-over-ranks device time).

    On one GPU the whole step is captured once as a CUDA graph and replayed
    (a CIFAR-size step is ~300 small kernels, so eager launches make it host
    bound); the warm-up runs on the capture stream so every per-stream
    resource of the SCC plans exists before capture.  Under torchrun (DDP)
    the step runs eagerly."""
    dev = torch.device("cuda", torch.cuda.current_device())
    ws = dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1
    torch.manual_seed(seed)
    model = MODELS[model_name](num_classes=num_classes, device=dev)
    if ws > 1:
        model = nn.parallel.DistributedDataParallel(model, device_ids=[dev.index])
    opt = torch.optim.SGD(model.parameters(), lr=0.05, momentum=0.9, weight_decay=5e-4)
    gen = torch.Generator(device=dev).manual_seed(seed + (dist.get_rank() if ws > 1 else 0))
    x = torch.randn(batch, 3, image, image, device=dev, generator=gen)
    y = torch.randint(0, num_classes, (batch,), device=dev, generator=gen)
    loss_fn = nn.CrossEntropyLoss()

    def step():
        opt.zero_grad(set_to_none=True)
        loss = loss_fn(model(x), y)
        loss.backward()
        opt.step()
        return loss

    launch = "eager"
    stream = torch.cuda.Stream(dev)
    stream.wait_stream(torch.cuda.current_stream(dev))
    with torch.cuda.stream(stream):
        losses = [float(step().item()) for _ in range(max(warmup, 1))]
        run = step
        if graph and ws == 1:
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
            "launch": launch,
            "data": "synthetic N(0,1) images, uniform labels"}
