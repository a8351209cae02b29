"""Diagnostic: epilogue store throughput vs output allocation type."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
rt = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
def cuda_malloc(nbytes):
    p = C.c_void_p(); assert rt.cudaMalloc(C.byref(p), C.c_size_t(nbytes)) == 0; return p.value
cfg = scc.scc_config_new(64, 128, 2, "50%", True); cfg.set_path(2)
x = torch.randn(32, 64, 32, 32, device="cuda"); wts = scc.scc_weights_init(cfg)
L = _lib.lib(); s = torch.cuda.current_stream().cuda_stream
y_t = torch.empty(32, 128, 32, 32, device="cuda")
y_raw = cuda_malloc(y_t.numel() * 4)
buf = (C.c_uint64 * 32)()
def run(yp):
    _lib.check(L.scc_forward_f32(cfg.handle, 32, 32, 32, x.data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), yp, s))
for name, yp in (("torch.empty", y_t.data_ptr()), ("cudaMalloc", y_raw)):
    for _ in range(5): run(yp)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(); [run(yp) for _ in range(50)]; e1.record(); e1.synchronize()
    run(yp); torch.cuda.synchronize(); L.scc_debug_trace(buf, 32)
    print(f"{name}: fwd {1e3*e0.elapsed_time(e1)/50:.1f} us/call; tile0 mma->epi {(buf[7]-buf[6])/1e3:.2f} us")
# raw write bandwidth into each buffer
z = torch.randn(y_t.numel(), device="cuda")
for name in ("torch", "raw"):
    if name == "torch":
        dst = y_t.view(-1)
    else:
        continue
    torch.cuda.synchronize(); e0.record()
    for _ in range(50): dst.copy_(z)
    e1.record(); e1.synchronize()
    print(f"copy into {name}: {2*z.numel()*4/(e0.elapsed_time(e1)/50*1e-3)/1e9:.0f} GB/s")
print("PYTORCH_CUDA_ALLOC_CONF", os.environ.get("PYTORCH_CUDA_ALLOC_CONF"))
