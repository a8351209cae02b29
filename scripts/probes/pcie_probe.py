"""PCIe ceiling for the host-buffer entry points: pinned H2D and D2H of the
config-1 step's bytes (25.2 MB each way), alone and concurrently on two
streams, plus scc_fwd_bwd_host_f32 at 1..8 chunks."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
torch.cuda.set_device(0)
nb = 25182720 // 4
h1 = torch.randn(nb).pin_memory(); h2 = torch.empty(nb).pin_memory()
d1 = torch.empty(nb, device="cuda"); d2 = torch.randn(nb, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, it=20):
    fn(); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(it): fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / it * 1e3
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
def both():
    h2d(); d2h()
r = {"h2d_ms": t(h2d), "d2h_ms": t(d2h), "both_ms": t(both)}
r["h2d_GBs"] = round(nb * 4 / r["h2d_ms"] / 1e6, 1); r["d2h_GBs"] = round(nb * 4 / r["d2h_ms"] / 1e6, 1)
print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in r.items()}))
