"""Practical HBM floor at the config-1 backward's byte count: one fused
elementwise kernel reading 25.2 MB (dy + x) and writing 8.4 MB (dx), the same
8-buffer-set rotation and 16-call CUDA graphs as scripts/bwd_timing.py."""
import torch
R, N, CI, CO, P = 8, 32, 64, 128, 1024
xs = [torch.randn(N, CI, P, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, P, device="cuda") for _ in range(R)]
dxs = [torch.empty(N, CI, P, device="cuda") for _ in range(R)]
def t(name, fn, nbytes):
    for i in range(R): fn(i)
    torch.cuda.synchronize()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(16): fn(k % R)
        g.replay(); st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10): g.replay()
        e1.record(st); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 160
    print(f"{name}: {us:.2f} us per call, {nbytes / us / 1e3:.0f} GB/s", flush=True)
t("addcmul dx = x + dy[:, :64] * dy[:, 64:] (33.6 MB)", lambda i: torch.addcmul(xs[i], dys[i][:, :CI], dys[i][:, CI:], out=dxs[i]), 4 * N * P * 4 * CI)
t("add dx = x + x' (25.2 MB)", lambda i: torch.add(xs[i], xs[(i + 1) % R], out=dxs[i]), 4 * N * P * 3 * CI)
t("copy dy -> dy' (33.6 MB)", lambda i: dys[(i + 1) % R].copy_(dys[i]), 4 * N * P * 2 * CO)
