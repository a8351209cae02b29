import os, sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
torch.cuda.set_device(0)
n, ci, co, h, w = 32, 64, 128, 32, 32
cfg = scc.scc_config_new(ci, co, 2, "50%", True)
xh = torch.randn(n, ci, h, w).pin_memory(); dyh = torch.randn(n, co, h, w).pin_memory()
yh = torch.empty(n, co, h, w).pin_memory(); dxh = torch.empty(n, ci, h, w).pin_memory()
xd = torch.empty(n, ci, h, w, device="cuda"); dyd = torch.empty(n, co, h, w, device="cuda")
yd = torch.empty(n, co, h, w, device="cuda"); dxd = torch.empty(n, ci, h, w, device="cuda")
wts = scc.scc_weights_init(cfg)
s_in, s_c, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def run(k, copies_only=False):
    m = n // k
    evs = []
    for i in range(k):
        sl = slice(i * m, (i + 1) * m)
        with torch.cuda.stream(s_in):
            xd[sl].copy_(xh[sl], non_blocking=True); dyd[sl].copy_(dyh[sl], non_blocking=True)
            e = torch.cuda.Event(); e.record(s_in)
        s_c.wait_event(e)
        if not copies_only:
            sp = s_c.cuda_stream
            _lib.check(L.scc_forward_f32(cfg.handle, m, h, w, xd[sl].data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), yd[sl].data_ptr(), sp))
            _lib.check(L.scc_backward_data_f32(cfg.handle, m, h, w, dyd[sl].data_ptr(), wts.weight.data_ptr(), dxd[sl].data_ptr(), sp))
        e2 = torch.cuda.Event(); e2.record(s_c)
        s_out.wait_event(e2)
        with torch.cuda.stream(s_out):
            yh[sl].copy_(yd[sl], non_blocking=True); dxh[sl].copy_(dxd[sl], non_blocking=True)
    torch.cuda.synchronize()
for k in (1, 2, 4, 8):
    for co_ in (True, False):
        run(k, co_)
        t0 = time.perf_counter()
        for _ in range(20): run(k, co_)
        print(k, "copies_only" if co_ else "with_kernels", round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms", flush=True)

# variant: x / dy (and y / dx) copies on separate streams (more copy engines)
s_in2, s_out2 = torch.cuda.Stream(), torch.cuda.Stream()
def run2(k):
    m = n // k
    for i in range(k):
        sl = slice(i * m, (i + 1) * m)
        with torch.cuda.stream(s_in):
            xd[sl].copy_(xh[sl], non_blocking=True)
            e = torch.cuda.Event(); e.record(s_in)
        with torch.cuda.stream(s_in2):
            dyd[sl].copy_(dyh[sl], non_blocking=True)
            e1 = torch.cuda.Event(); e1.record(s_in2)
        s_c.wait_event(e); s_c.wait_event(e1)
        e2 = torch.cuda.Event(); e2.record(s_c)
        s_out.wait_event(e2); s_out2.wait_event(e2)
        with torch.cuda.stream(s_out):
            yh[sl].copy_(yd[sl], non_blocking=True)
        with torch.cuda.stream(s_out2):
            dxh[sl].copy_(dxd[sl], non_blocking=True)
    torch.cuda.synchronize()
for k in (2, 4, 8):
    run2(k)
    t0 = time.perf_counter()
    for _ in range(20): run2(k)
    print(k, "copies_only 4 streams", round((time.perf_counter() - t0) / 20 * 1e3, 3), "ms", flush=True)
