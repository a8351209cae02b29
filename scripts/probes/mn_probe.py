"""MN-major kind::tf32 probe driver (tests/cuda/mn_probe.cu): which LBO/SBO
assignment makes a TMA SWIZZLE_128B_ATOM_32B tile a valid MN-major operand."""
import ctypes as C, os, sys
import numpy as np, torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "mn_probe.so"))
lib.mn_probe.argtypes = [C.c_void_p] * 3 + [C.c_int] * 3
def trunc(a):
    return (a.view(np.uint32) & np.uint32(0xFFFFE000)).view(np.float32).astype(np.float64)
rng = np.random.default_rng(0)
x = rng.standard_normal((64, 128)).astype(np.float32)
w = rng.standard_normal((128, 64)).astype(np.float32)
ref0 = trunc(x).T @ trunc(w).T     # [p][oc]
ref1 = ref0.T                      # [oc][p]
xt, wt = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
for mode in (0, 1):
    for lbo, sbo in ((8192, 512), (512, 8192), (8192, 1024), (1024, 8192)):
        out = torch.zeros(128, 128, device="cuda")
        rc = lib.mn_probe(xt.data_ptr(), wt.data_ptr(), out.data_ptr(), mode, lbo, sbo)
        got = out.cpu().numpy().astype(np.float64)
        ref = ref0 if mode == 0 else ref1
        err = np.abs(got - ref).max() / np.abs(ref).max()
        print(f"mode {mode} lbo {lbo} sbo {sbo}: rc {rc} err {err:.3e} nz {np.count_nonzero(got)}", flush=True)
