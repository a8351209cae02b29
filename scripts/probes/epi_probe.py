"""Epilogue cost probe (tests/cuda/epi_probe.cu): cycles per 32-column group."""
import ctypes as C, os
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "epi_probe.so"))
lib.epi_probe.argtypes = [C.c_void_p, C.c_int, C.c_int]
names = {0: "LDTM x32 + wait", 1: "LDTM + 32 STS", 2: "32 STS only", 3: "LDTM + 32 STS with MMAs running"}
for mode in (0, 1, 2, 3):
    for groups in (64,):
        out = torch.zeros(4, dtype=torch.int64, device="cuda")
        lib.epi_probe(out.data_ptr(), mode, groups)
        lib.epi_probe(out.data_ptr(), mode, groups)
        out.zero_(); lib.epi_probe(out.data_ptr(), mode, groups)
        o = out.cpu().tolist()
        print(f"mode {mode} ({names[mode]}): {o[0] / groups:.0f} cycles/group (4 warps concurrent), mmas {o[1]}", flush=True)
