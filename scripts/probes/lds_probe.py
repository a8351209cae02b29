"""Shared-memory latency / STS throughput probe (tests/cuda/lds_probe.cu)."""
import ctypes as C, os
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "lds_probe.so"))
lib.lds_probe.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int]
for smem in (65536, 226 * 1024):
    for mode in (0, 1):
        for busy in (0, 9):
            out = torch.zeros(4, dtype=torch.int64, device="cuda")
            lib.lds_probe(out.data_ptr(), busy, 1024, mode, smem); lib.lds_probe(out.data_ptr(), busy, 1024, mode, smem)
            print(f"smem {smem // 1024} KB {'LDS chase' if mode == 0 else 'STS'} busy {busy}: {out[0].item() / 1024:.1f} cycles/op", flush=True)
