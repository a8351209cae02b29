"""Panel-build micro-benchmark (tests/cuda/build_probe.cu)."""
import ctypes as C, os
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "build_probe.so"))
lib.build_probe.argtypes = [C.c_void_p, C.c_int, C.c_int]
for warm in (0, 1):
    for bwd, f4 in ((0, 0), (0, 1), (1, 0)):
        out = torch.zeros(4, dtype=torch.int64, device="cuda")
        lib.build_probe(out.data_ptr(), bwd, f4); out.zero_(); out[3] = warm; lib.build_probe(out.data_ptr(), bwd, f4)
        print(f"warm={warm} {'bwd' if bwd else 'fwd'} fwd4={f4} build: {out[0].item()} cycles", flush=True)
