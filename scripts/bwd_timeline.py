"""Timeline of one concurrent backward call (backward-data band kernel on one SM
half, backward-weight on the other): per-CTA start / end spreads of both
kernels from their %globaltimer traces, on a common clock."""
import ctypes as C, os, sys, statistics
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
N, CI, CO, H, W = 32, 64, 128, 32, 32
cfg = scc.scc_config_new(CI, CO, 2, "50%", True)
x = torch.randn(N, CI, H, W, device="cuda"); dy = torch.randn(N, CO, H, W, device="cuda")
y = torch.empty(N, CO, H, W, device="cuda"); dx = torch.empty_like(x)
wts = scc.scc_weights_init(cfg)
ws = torch.empty(cfg.workspace_bytes(N, H, W), dtype=torch.uint8, device="cuda")
g = torch.empty(CO * 32 + CO, device="cuda")
s = torch.cuda.current_stream().cuda_stream
def fwd():
    _lib.check(L.scc_forward_f32(cfg.handle, N, H, W, x.data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), y.data_ptr(), s))
def bwd():
    _lib.check(L.scc_backward_f32(cfg.handle, N, H, W, dy.data_ptr(), x.data_ptr(), wts.weight.data_ptr(), dx.data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * 32, ws.data_ptr(), ws.numel(), s))
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    s = st.cuda_stream
    for _ in range(5):
        fwd(); bwd()
    st.synchronize()
    gf = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gf, stream=st):
        fwd()
    gb = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gb, stream=st):
        bwd()
torch.cuda.synchronize()
for _ in range(3):
    gf.replay(); gb.replay()
torch.cuda.synchronize()
gf.replay(); torch.cuda.synchronize()
n = 128 + 64 + 2048 + 64 + 3 * 256
buf = (C.c_uint64 * n)()
L.scc_debug_trace(buf, n)
f_st = [buf[192 + 2 * i] for i in range(148)]; f_en = [buf[193 + 2 * i] for i in range(148)]
gb.replay(); torch.cuda.synchronize()
L.scc_debug_trace(buf, n)
b_st = [buf[192 + 2 * i] for i in range(74)]; b_en = [buf[193 + 2 * i] for i in range(74)]
base = 128 + 64 + 2048 + 64
w_st = [buf[base + 3 * i] for i in range(74)]; w_af = [buf[base + 3 * i + 1] for i in range(74)]; w_ba = [buf[base + 3 * i + 2] for i in range(74)]
w_end = buf[128 + 64 + 2048 + 37]
t0 = min(b_st + w_st)
def spread(name, v, ref):
    d = sorted((x - ref) / 1e3 for x in v)
    print(f"  {name:28s} min {d[0]:6.2f} med {statistics.median(d):6.2f} max {d[-1]:6.2f} us")
print("forward (148 CTAs), relative to its first CTA start:")
spread("CTA start", f_st, min(f_st)); spread("epilogue end", f_en, min(f_st))
print("concurrent backward, relative to the first CTA start of either kernel:")
spread("dx CTA start", b_st, t0); spread("dx epilogue end", b_en, t0)
spread("dW CTA start", w_st, t0); spread("dW mainloop end", w_af, t0); spread("dW barrier arrive", w_ba, t0)
print(f"  dW CTA0 end {(w_end - t0) / 1e3:.2f} us")
