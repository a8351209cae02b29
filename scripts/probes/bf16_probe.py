"""kind::f16 (bf16) operand conventions and issue rate (tests/cuda/bf16_probe.cu)."""
import ctypes as C, os
import numpy as np
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "bf16_probe.so"))
M, N, K = 128, 64, 128
rng = np.random.default_rng(0)
a = rng.standard_normal((M, K)).astype(np.float32)
b = rng.standard_normal((K, N)).astype(np.float32)
bf = lambda v: torch.from_numpy(v).to(torch.bfloat16).float().numpy().astype(np.float64)
ref = bf(a) @ bf(b)
at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
out = torch.zeros(M, N, device="cuda")
for mode in (0, 1):
    for swap in (0, 1):
        for lbo, sbo in ((8192, 1024), (16, 1024)) if mode == 0 else ((16, 1024),):
            out.zero_()
            rc = lib.bf16_probe(C.c_void_p(at.data_ptr()), C.c_void_p(bt.data_ptr()), C.c_void_p(out.data_ptr()), mode, swap, lbo, sbo)
            o = out.cpu().numpy().astype(np.float64)
            err = np.max(np.abs(o - ref)) / np.max(np.abs(ref))
            print(f"mode {mode} ({'B MN-major' if mode == 0 else 'B K-major'}) swap {swap} lbo {lbo} sbo {sbo}: rc {rc} err {err:.3e}", flush=True)
res = torch.zeros(148, dtype=torch.int64, device="cuda")
for m in (128, 64):
  for b_mn in (1, 0):
    row = []
    for n in (32, 64, 128, 256):
        reps = 512
        assert lib.bf16_rate(m, n, b_mn, reps, 148, C.c_void_p(res.data_ptr())) == 0
        v = sorted(res.tolist())
        row.append(f"N={n}: {v[74] / reps:6.1f}")
    print(f"bf16 TS M={m} K=16 B {'MN' if b_mn else 'K '}-major  " + "  ".join(row) + "  cycles/MMA", flush=True)
