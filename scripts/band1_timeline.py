"""Generation-1 band kernel (scc_tc.cu, forward): CTA-0 %globaltimer timeline
of one call at a sweep shape ($SCC_SHAPE = "ci,co,cg,ov%,n,h,w", default C256
56x56 cg2 co50): setup, first TMA, first stage landed / converted, per-tile
MMA commit and epilogue done."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
f = os.environ.get("SCC_SHAPE", "256,256,2,50%,32,56,56").split(",")
CI, CO, CG, OV, N, H, W = int(f[0]), int(f[1]), int(f[2]), f[3], int(f[4]), int(f[5]), int(f[6])
cfg = scc.scc_config_new(CI, CO, CG, OV, True)
x = torch.randn(N, CI, H, W, device="cuda")
dy = torch.randn(N, CO, H, W, device="cuda")
wts = scc.scc_weights_init(cfg)
for _ in range(3):  # OP=bdata: backward-data (the same kernel, bf16x3)
    y = scc.scc_backward_input(dy, wts, cfg) if os.environ.get("OP") == "bdata" else scc.scc_forward(x, wts, cfg)
torch.cuda.synchronize()
buf = (C.c_uint64 * 32)()
L.scc_debug_trace(buf, 32)
t = [buf[i] for i in range(32)]
t0 = t[0]
if t0 == 0:
    sys.exit("no trace: build with make -C paper_2101_00745_b200/csrc SCC_EXTRA=-DSCC_TRACE and load it via SCC_LIB_PATH")
lab = {0: "start", 1: "setup", 2: "p_first_tma", 3: "p_dep", 4: "conv_first_landed", 5: "mma_first_conv", 30: "end"}
for i in range(8):
    lab[6 + 2 * i] = f"mma_commit{i}"; lab[7 + 2 * i] = f"epi_done{i}"
print(" ".join(f"{lab[i]}={(t[i] - t0) / 1e3:.2f}" for i in sorted(lab) if t[i] >= t0 and t[i] - t0 < 1e8))
