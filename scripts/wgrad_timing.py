"""Backward-weight per-call device time (graph of 20 calls, inputs rotated over
8 buffer sets) for each tensor-core generation, plus the gen-2 CTA-0 timeline."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
N, CI, CO, H, W, CG = 32, 64, 128, 32, 32, 2
cfg = scc.scc_config_new(CI, CO, CG, "50%", True)
R = 8
xs = [torch.randn(N, CI, H, W, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, H, W, device="cuda") for _ in range(R)]
ws = torch.empty(cfg.workspace_bytes(N, H, W), dtype=torch.uint8, device="cuda")
dw = torch.empty(CO * 32, device="cuda"); db = torch.empty(CO, device="cuda")
def bw(i, s):
    _lib.check(L.scc_backward_weight_f32(cfg.handle, N, H, W, dys[i].data_ptr(), xs[i].data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(), s))
for path, name in ((_lib.SCC_PATH_TENSOR_STREAMED, "gen1"), (_lib.SCC_PATH_TENSOR, "gen2")):
    cfg.set_path(path)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for i in range(R): bw(i, st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(20): bw(k % R, st.cuda_stream)
        g.replay(); st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10): g.replay()
        e1.record(st); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / 200
    print(f"{name} bwd_weight: {us:.2f} us/call  {4 * N * H * W * (CI + CO) / us / 1e3:.0f} GB/s", flush=True)
bw(0, torch.cuda.current_stream().cuda_stream); torch.cuda.synchronize()
n = 128 + 64 + 2048 + 64 + 3 * 256
buf = (C.c_uint64 * n)()
L.scc_debug_trace(buf, n)
t = [buf[128 + 64 + 2048 + i] for i in range(64)]
t0 = t[0]
lab = {0: "start", 1: "dep", 34: "accfull", 35: "partials", 36: "gbar", 37: "end", 40: "p_loop", 41: "p_free", 42: "p_expect", 43: "p_tma_first", 44: "p_dy_done"}
for i in range(8):
    lab[2 + i] = f"tma{i}"; lab[10 + i] = f"mma{i}"; lab[18 + i] = f"full{i}"; lab[26 + i] = f"conv{i}"
print("gen2", " ".join(f"{lab[i]}={(t[i] - t0) / 1e3:.2f}" for i in sorted(lab) if t[i] >= t0 and t[i] - t0 < 1e8))

import statistics
base = 128 + 64 + 2048 + 64
st = [buf[base + 3 * i] for i in range(148)]; af = [buf[base + 3 * i + 1] for i in range(148)]; ba = [buf[base + 3 * i + 2] for i in range(148)]
m0 = min(st)
f = lambda v: sorted((x - m0) / 1e3 for x in v)
for name, v in (("start", st), ("accfull", af), ("barrier arrive", ba)):
    d = f(v); print(f"{name}: min {d[0]:.2f} med {statistics.median(d):.2f} p90 {d[int(0.9 * len(d))]:.2f} max {d[-1]:.2f}")
