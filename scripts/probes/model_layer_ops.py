"""Per-op device time (CUDA graphs of 16 calls, 4 rotating sets) of every SCC
layer shape of SCC-ResNet-18 (CIFAR, batch 128; DW(stride) then SCC on the
output plane): forward, backward (scc_backward_f32), GB/s of the compulsory
bytes, and the kernel family AUTO picks."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
N = int(os.environ.get("BATCH", "128"))
SHAPES = [(64, 64, 32), (64, 128, 16), (128, 128, 16), (128, 256, 8), (256, 256, 8), (256, 512, 4), (512, 512, 4)]
def tg(f, R):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(R): f(i, st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(16): f(k % R, st.cuda_stream)
        g.replay(); st.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(10): g.replay()
        b.record(st); b.synchronize()
    return a.elapsed_time(b) * 1e3 / 160
tot = 0
for ci, co, hw in SHAPES:
    cfg = scc.scc_config_new(ci, co, 2, "50%", True)
    gw = cfg.group_width
    R = 4
    xs = [torch.randn(N, ci, hw, hw, device="cuda") for _ in range(R)]
    dys = [torch.randn(N, co, hw, hw, device="cuda") for _ in range(R)]
    ys = [torch.empty(N, co, hw, hw, device="cuda") for _ in range(R)]
    dxs = [torch.empty(N, ci, hw, hw, device="cuda") for _ in range(R)]
    wts = scc.scc_weights_init(cfg)
    g = torch.empty(co * gw + co, device="cuda")
    wsb = cfg.workspace_bytes(N, hw, hw)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    fwd = lambda i, s: _lib.check(L.scc_forward_f32(cfg.handle, N, hw, hw, xs[i].data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), ys[i].data_ptr(), s))
    bwd = lambda i, s: _lib.check(L.scc_backward_f32(cfg.handle, N, hw, hw, dys[i].data_ptr(), xs[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * co * gw, ws.data_ptr(), wsb, s))
    bd = lambda i, s: _lib.check(L.scc_backward_data_f32(cfg.handle, N, hw, hw, dys[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), s))
    bw = lambda i, s: _lib.check(L.scc_backward_weight_f32(cfg.handle, N, hw, hw, dys[i].data_ptr(), xs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * co * gw, ws.data_ptr(), wsb, s))
    tf, tb = tg(fwd, R), tg(bwd, R)
    tbd, tbw = tg(bd, R), tg(bw, R)
    P = hw * hw
    bf, bb = 4 * N * P * (ci + co), 4 * N * P * (2 * ci + co)
    tot += tf + tb
    print(f"{ci:4d}->{co:4d} {hw:2d}x{hw:<2d} path {cfg.path_for(N, hw, hw)}  fwd {tf:7.2f} us ({bf / tf / 1e3:6.0f} GB/s)  bwd {tb:7.2f} us ({bb / tb / 1e3:6.0f} GB/s)  [data {tbd:6.2f}  weight {tbw:6.2f}]", flush=True)
print(f"sum {tot:.1f} us")
