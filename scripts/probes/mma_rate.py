"""tcgen05.mma kind::tf32 issue rate per layout (tests/cuda/mma_rate_probe.cu):
cycles per MMA, M=128 K=8, for N in 32..256, A in TMEM or SMEM, B MN- or
K-major; one CTA per SM, median over CTAs."""
import ctypes as C, os, subprocess, sys
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
so = os.path.join(HERE, "tests", "cuda", "_build", "mma_rate_probe.so")
lib = C.CDLL(so)
out = torch.zeros(148, dtype=torch.int64, device="cuda")
for m, ts, b_mn, noise in ((128, 1, 1, 0), (128, 1, 0, 0), (128, 0, 1, 0), (128, 0, 0, 0), (64, 1, 1, 0), (128, 1, 1, 1), (128, 1, 1, 4)):
    if True:
        row = []
        for n in (32, 64, 128, 256):
            reps = 512
            assert lib.mma_rate(m, n, ts, b_mn, reps, 148, noise, C.c_void_p(out.data_ptr())) == 0
            v = sorted(out.tolist())
            row.append(f"N={n}: {v[74] / reps:6.1f}")
        print(f"noise={noise} M={m} {'TS' if ts else 'SS'} B {'MN' if b_mn else 'K '}-major  " + "  ".join(row) + "  cycles/MMA", flush=True)
