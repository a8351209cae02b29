"""Host vs device time per C-ABI call (diagnostic)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
path = int(sys.argv[1]) if len(sys.argv) > 1 else 2
cfg = scc.scc_config_new(64, 128, 2, "50%", True); cfg.set_path(path)
x = torch.randn(32, 64, 32, 32, device="cuda"); dy = torch.randn(32, 128, 32, 32, device="cuda")
wts = scc.scc_weights_init(cfg); y = torch.empty(32, 128, 32, 32, device="cuda"); dx = torch.empty_like(x)
L = _lib.lib(); s = torch.cuda.current_stream().cuda_stream
def fwd(): _lib.check(L.scc_forward_f32(cfg.handle, 32, 32, 32, x.data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), y.data_ptr(), s))
def bwdd(): _lib.check(L.scc_backward_data_f32(cfg.handle, 32, 32, 32, dy.data_ptr(), wts.weight.data_ptr(), dx.data_ptr(), s))
for name, f in (("fwd", fwd), ("bwd_data", bwdd)):
    for _ in range(5): f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(50): f()
    t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [f() for _ in range(50)]; e1.record(); e1.synchronize()
    # graph
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        s_saved = s
    print(f"{name}: host {1e6*(t1-t0)/50:.1f} us/call, host+drain {1e6*(t2-t0)/50:.1f} us/call, events {1e3*e0.elapsed_time(e1)/50:.1f} us/call")
import ctypes as _C
buf = (_C.c_uint64 * 32)()
for name, f in (("fwd", fwd), ("bwd_data", bwdd)):
    f(); torch.cuda.synchronize()
    n = L.scc_debug_trace(buf, 32)
    t0 = buf[0]
    lab = {0:"start",1:"setup",2:"prod_first_tma",3:"dep_ok",4:"conv_first_full",5:"mma_first_conv",30:"end"}
    for i in range(8): lab[6+2*i] = f"mma_commit_t{i}"; lab[7+2*i] = f"epi_done_t{i}"
    print(name, " ".join(f"{lab[i]}={(buf[i]-t0)/1e3:.2f}" for i in sorted(lab) if buf[i] >= t0 and buf[i]-t0 < 1e9))
ws = torch.empty(cfg.workspace_bytes(32, 32, 32), dtype=torch.uint8, device="cuda")
dw = torch.empty(128 * 32, device="cuda"); db = torch.empty(128, device="cuda")
def bwdw(): _lib.check(L.scc_backward_weight_f32(cfg.handle, 32, 32, 32, dy.data_ptr(), x.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(), s))
for _ in range(5): bwdw()
torch.cuda.synchronize()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(); [bwdw() for _ in range(50)]; e1.record(); e1.synchronize()
print(f"bwd_weight events {1e3*e0.elapsed_time(e1)/50:.1f} us/call")
buf64 = (_C.c_uint64 * 64)()
L.scc_debug_trace(buf64, 64)
w = [buf64[32 + i] for i in range(32)]
t0 = w[0]
print("wgrad: setup", (w[1]-t0)/1e3, "issue", [round((w[2+i]-t0)/1e3,2) for i in range(8)], "conv", [round((w[10+i]-t0)/1e3,2) for i in range(8)], "mma", [round((w[18+i]-t0)/1e3,2) for i in range(8)], "epi", (w[26]-t0)/1e3, "chunk1 prod: start/afree/A/tfree/B", [round((w[i]-t0)/1e3, 2) for i in (27, 28, 29, 30, 31)])
