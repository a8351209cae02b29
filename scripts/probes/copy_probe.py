"""What does a plain device copy of the config-1 sizes achieve (the same
rotation over 8 buffer sets as the SCC timings)?"""
import torch
R = 8
N, CI, CO, P = 32, 64, 128, 1024
xs = [torch.randn(N, CI, P, device="cuda") for _ in range(R)]
ys = [torch.empty(N, CO, P, device="cuda") for _ in range(R)]
big = [torch.randn(N, CO, P, device="cuda") for _ in range(R)]
def t(name, fn, nbytes):
    for i in range(R): fn(i)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for k in range(16): fn(k % R)
    g.replay(); torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): g.replay()
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 160
    print(f"{name}: {us:.2f} us  {nbytes / us / 1e3:.0f} GB/s", flush=True)
t("copy 16.8 MB -> 16.8 MB", lambda i: ys[i].copy_(big[i]), 2 * 4 * N * CO * P)
t("x (8.4 MB) -> y (16.8 MB) as [x, x]", lambda i: ys[i].view(N, 2, CI, P).copy_(xs[i].view(N, 1, CI, P).expand(N, 2, CI, P)), 4 * N * (CI + CO) * P)
t("read 16.8 + read 8.4 (sum)", lambda i: torch.add(big[i][:, :CI], xs[i], out=xs[(i + 1) % R]), 4 * N * P * 3 * CI)
