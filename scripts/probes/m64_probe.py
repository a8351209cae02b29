"""M = 64 kind::f16 MMA: which TMEM lanes hold D (A and D at lane base 0 or
64), tests/cuda/bf16_probe.cu m64_probe."""
import ctypes as C, os
import numpy as np
import torch
HERE = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
lib = C.CDLL(os.path.join(HERE, "tests", "cuda", "_build", "bf16_probe.so"))
rng = np.random.default_rng(0)
a = rng.standard_normal((64, 128)).astype(np.float32)
b = rng.standard_normal((128, 64)).astype(np.float32)
bf = lambda v: torch.from_numpy(v).to(torch.bfloat16).double().numpy()
ref = bf(a) @ bf(b)
at, bt = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
out = torch.zeros(128, 64, device="cuda")
for lb in (0, 64, 32, -1):
    rc = lib.m64_probe(C.c_void_p(at.data_ptr()), C.c_void_p(bt.data_ptr()), C.c_void_p(out.data_ptr()), lb)
    o = out.cpu().numpy().astype(np.float64)
    written = [i for i in range(128) if not np.all(o[i] == 7777.0)]
    print(f"lane base {lb}: rc {rc}; lanes written: {written[:4]}..{written[-4:] if written else []} ({len(written)})")
    if len(written) == 64:
        got = o[written]  # lanes ascending = rows 0..63 when lane = (r % 16) + 32 (r / 16)
        print("   err vs bf16 product rows 0..63 in lane order:", np.abs(got - ref).max() / np.abs(ref).max())
