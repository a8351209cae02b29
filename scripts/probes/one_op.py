"""Run one SCC op a few times on config 1 or $SCC_SHAPE (for ncu captures).
usage: one_op.py fwd|bwd_data|bwd_weight|bwd [path]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
op = sys.argv[1]
path = int(sys.argv[2]) if len(sys.argv) > 2 else _lib.SCC_PATH_TENSOR
N, CI, CO, H, W = 32, 64, 128, 32, 32
CG, OV = 2, "50%"
if os.environ.get("SCC_SHAPE"):  # "ci,co,cg,ov%,n,h,w"
    f = os.environ["SCC_SHAPE"].split(",")
    CI, CO, CG, OV, N, H, W = int(f[0]), int(f[1]), int(f[2]), f[3], int(f[4]), int(f[5]), int(f[6])
cfg = scc.scc_config_new(CI, CO, CG, OV, True); cfg.set_path(path)
L = _lib.lib(); s = torch.cuda.current_stream().cuda_stream
x = torch.randn(N, CI, H, W, device="cuda"); dy = torch.randn(N, CO, H, W, device="cuda")
y = torch.empty(N, CO, H, W, device="cuda"); dx = torch.empty_like(x)
wts = scc.scc_weights_init(cfg)
ws = torch.empty(max(cfg.workspace_bytes(N, H, W), 16), dtype=torch.uint8, device="cuda")
dw = torch.empty(CO * cfg.group_width, device="cuda"); db = torch.empty(CO, device="cuda")
for _ in range(4):
    if op in ("fwd",):
        _lib.check(L.scc_forward_f32(cfg.handle, N, H, W, x.data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), y.data_ptr(), s))
    if op in ("bwd_data",):
        _lib.check(L.scc_backward_data_f32(cfg.handle, N, H, W, dy.data_ptr(), wts.weight.data_ptr(), dx.data_ptr(), s))
    if op in ("bwd_weight",):
        _lib.check(L.scc_backward_weight_f32(cfg.handle, N, H, W, dy.data_ptr(), x.data_ptr(), dw.data_ptr(), db.data_ptr(), ws.data_ptr(), ws.numel(), s))
torch.cuda.synchronize()
print("ok")
