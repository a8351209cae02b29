"""Per-op device time (16-call CUDA graphs, 4 rotating sets) at a sweep shape,
for launch-list profiling under ncu.  SCC_SHAPE=ci,co,cg,ov,n,h,w  OPS=fwd,bdata,bwt"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
f = os.environ.get("SCC_SHAPE", "256,256,2,50%,32,14,14").split(",")
CI, CO, CG, OV, N, H, W = int(f[0]), int(f[1]), int(f[2]), f[3], int(f[4]), int(f[5]), int(f[6])
cfg = scc.scc_config_new(CI, CO, CG, OV, True)
gw = cfg.group_width
R = 4
xs = [torch.randn(N, CI, H, W, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, H, W, device="cuda") for _ in range(R)]
ys = [torch.empty(N, CO, H, W, device="cuda") for _ in range(R)]
dxs = [torch.empty(N, CI, H, W, device="cuda") for _ in range(R)]
wts = scc.scc_weights_init(cfg)
g = torch.empty(CO * gw + CO, device="cuda")
wsb = cfg.workspace_bytes(N, H, W)
ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
ops = {
    "fwd": lambda i, s: L.scc_forward_f32(cfg.handle, N, H, W, xs[i].data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), ys[i].data_ptr(), s),
    "bdata": lambda i, s: L.scc_backward_data_f32(cfg.handle, N, H, W, dys[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), s),
    "bwt": lambda i, s: L.scc_backward_weight_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * gw, ws.data_ptr(), wsb, s),
}
sel = os.environ.get("OPS", "fwd,bdata,bwt").split(",")
st = torch.cuda.Stream()
for name in sel:
    f_ = ops[name]
    with torch.cuda.stream(st):
        for i in range(R): _lib.check(f_(i, st.cuda_stream))
        st.synchronize()
        if os.environ.get("EAGER"):
            for i in range(4): _lib.check(f_(i % R, st.cuda_stream))
            st.synchronize()
            continue
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for k in range(16): _lib.check(f_(k % R, st.cuda_stream))
        gr.replay(); st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10): gr.replay()
        e1.record(st); e1.synchronize()
    print(f"{name}: {e0.elapsed_time(e1) * 1e3 / 160:.2f} us per call", flush=True)
