"""Device time per CUDA-graph replay of: forward only, backward only (the
concurrent scc_backward_f32), forward+backward -- config 1, inputs rotated
over 8 buffer sets."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
N, CI, CO, H, W = 32, 64, 128, 32, 32
cfg = scc.scc_config_new(CI, CO, 2, "50%", True)
R = 8
xs = [torch.randn(N, CI, H, W, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, H, W, device="cuda") for _ in range(R)]
ys = [torch.empty(N, CO, H, W, device="cuda") for _ in range(R)]
dxs = [torch.empty(N, CI, H, W, device="cuda") for _ in range(R)]
wts = scc.scc_weights_init(cfg)
ws = torch.empty(cfg.workspace_bytes(N, H, W), dtype=torch.uint8, device="cuda")
g = torch.empty(CO * 32 + CO, device="cuda")
def fwd(i, s):
    _lib.check(L.scc_forward_f32(cfg.handle, N, H, W, xs[i].data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), ys[i].data_ptr(), s))
def bwd(i, s):
    _lib.check(L.scc_backward_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * 32, ws.data_ptr(), ws.numel(), s))
def both(i, s):
    fwd(i, s); bwd(i, s)
def bdata(i, s):
    _lib.check(L.scc_backward_data_f32(cfg.handle, N, H, W, dys[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), s))
def bweight(i, s):
    _lib.check(L.scc_backward_weight_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * 32, ws.data_ptr(), ws.numel(), s))
st = torch.cuda.Stream()
for name, f in (("fwd", fwd), ("bwd", bwd), ("fwd+bwd", both), ("bwd_data", bdata), ("bwd_weight", bweight)):
    with torch.cuda.stream(st):
        for i in range(R): f(i, st.cuda_stream)
        st.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for k in range(16): f(k % R, st.cuda_stream)
        gr.replay(); st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10): gr.replay()
        e1.record(st); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 1e3 / 160:.2f} us per call", flush=True)
