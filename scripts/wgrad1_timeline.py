"""Generation-1 backward-weight kernel (scc_tc_wgrad.cu): CTA-0 %globaltimer
timeline of one call at a sweep shape ($SCC_SHAPE = "ci,co,cg,ov%,n,h,w",
default C256 56x56 cg2 co50): chunk i issued (producer), converted (dy
converters), MMA committed, epilogue done."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
f = os.environ.get("SCC_SHAPE", "256,256,2,50%,32,56,56").split(",")
CI, CO, CG, OV, N, H, W = int(f[0]), int(f[1]), int(f[2]), f[3], int(f[4]), int(f[5]), int(f[6])
cfg = scc.scc_config_new(CI, CO, CG, OV, True)
x = torch.randn(N, CI, H, W, device="cuda"); dy = torch.randn(N, CO, H, W, device="cuda")
ws = torch.empty(cfg.workspace_bytes(N, H, W), dtype=torch.uint8, device="cuda")
dw = torch.empty(CO * cfg.group_width, device="cuda"); db = torch.empty(CO, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.check(L.scc_backward_weight_f32(cfg.handle, N, H, W, dy.data_ptr(), x.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(), s))
torch.cuda.synchronize()
buf = (C.c_uint64 * 64)()
L.scc_debug_trace(buf, 64)
t = [buf[32 + i] for i in range(32)]
t0 = t[0]
if t0 == 0:
    sys.exit("no trace: build with make -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE and load it via SCC_LIB_PATH")
lab = {0: "start", 1: "setup", 26: "epi_done", 27: "p_wait_afree", 28: "p_afree_ok", 29: "p_dy_issued", 30: "p_tfree_ok", 31: "p_x_issued"}
for i in range(8):
    lab[2 + i] = f"issued{i}"; lab[10 + i] = f"conv{i}"; lab[18 + i] = f"mma{i}"
print(" ".join(f"{lab[i]}={(t[i] - t0) / 1e3:.2f}" for i in sorted(lab) if t[i] >= t0 and t[i] - t0 < 1e8))
