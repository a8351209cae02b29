"""Fused backward kernel (scc_tc_bwd.cu) timeline: per-call device time of
scc_backward_f32 / backward-data / backward-weight (graphs of 16 calls, inputs
rotated over 8 buffer sets), then the CTA-0 %globaltimer slots and the per-CTA
start / end spread of one call.  Needs a -DSCC_TRACE build for the timeline
(make -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE)."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
N, CI, CO, H, W = 32, 64, 128, 32, 32
cfg = scc.scc_config_new(CI, CO, 2, "50%", True)
R = 8
xs = [torch.randn(N, CI, H, W, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, H, W, device="cuda") for _ in range(R)]
dxs = [torch.empty(N, CI, H, W, device="cuda") for _ in range(R)]
wts = scc.scc_weights_init(cfg)
ws = torch.empty(cfg.workspace_bytes(N, H, W), dtype=torch.uint8, device="cuda")
g = torch.empty(CO * 32 + CO, device="cuda")
def bwd(i, s):
    _lib.check(L.scc_backward_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * 32, ws.data_ptr(), ws.numel(), s))
def bdata(i, s):
    _lib.check(L.scc_backward_data_f32(cfg.handle, N, H, W, dys[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), s))
def bweight(i, s):
    _lib.check(L.scc_backward_weight_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), g.data_ptr(), g.data_ptr() + 4 * CO * 32, ws.data_ptr(), ws.numel(), s))
st = torch.cuda.Stream()
for name, f in (("bwd", bwd), ("bwd_data", bdata), ("bwd_weight", bweight)):
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
for name, f in (("bwd_data", bdata), ("bwd", bwd)):
    with torch.cuda.stream(st):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for k in range(4): f(k % R, st.cuda_stream)
        gr.replay(); st.synchronize()
    n = 128 + 512
    buf = (C.c_uint64 * n)()
    L.scc_debug_trace_fused(buf, n)
    t = [buf[i] for i in range(128)]
    t0 = t[48]
    print("raw", t[48:53], t[60:63])
    if t0 == 0:
        print("(no trace: build with SCC_EXTRA=-DSCC_TRACE)"); break
    lab = {48: "start", 49: "tmem", 50: "wt_ready", 51: "accfull", 52: "end", 53: "e_dep", 55: "e_bar", 60: "red_entry", 61: "red_dep", 62: "red_end", 59: "prev_red_end"}
    for k in range(8):
        lab[k] = f"tma{k}"
        if k < 4: lab[64 + k] = f"eld{k}"; lab[68 + k] = f"ewr{k}"; lab[72 + k] = f"eb1_{k}"; lab[76 + k] = f"eb2_{k}"; lab[80 + k] = f"eadd{k}"
        if k < 3: lab[56 + k] = f"xconv{k}"
        lab[k] = f"tma{k}"; lab[8 + k] = f"conv{k}"; lab[16 + k] = f"mdw{k}"; lab[24 + k] = f"mdx{k}"; lab[32 + k] = f"dxfull{k}"; lab[40 + k] = f"store{k}"  # k = block pair
    print(name, " ".join(f"{lab[i]}={(t[i] - t0) / 1e3:.2f}" for i in sorted(lab) if t[i] > 0 and abs(t[i] - t0) < 1e8))
    cs = [buf[128 + 2 * i] for i in range(148)]; ce = [buf[128 + 2 * i + 1] for i in range(148)]
    m0 = min(cs)
    s_ = sorted((x - m0) / 1e3 for x in cs); e_ = sorted((x - m0) / 1e3 for x in ce)
    print(f"  CTA start min/med/max {s_[0]:.2f}/{s_[74]:.2f}/{s_[-1]:.2f}  end {e_[0]:.2f}/{e_[74]:.2f}/{e_[-1]:.2f}")
    if os.environ.get("CTA_DUMP") and name == "bwd":
        for i in range(148):
            print(f"  cta {i:3d} sm {cs[i] & 0xFF:3d} start {((cs[i] & ~0xFF) - m0) / 1e3:6.2f} end {(ce[i] - m0) / 1e3:6.2f}")
