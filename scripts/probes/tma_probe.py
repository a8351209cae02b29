import ctypes as C, os, subprocess, sys, torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
so = os.path.join(root, "tests/cuda/_build/tma_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                           "-I" + os.path.join(root, "paper_2101_00745_b200/csrc"), "-o", so, os.path.join(root, "tests/cuda/tma_probe.cu")])
L = C.CDLL(so)
L.tma_probe.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
g = torch.randn(8192 * 1024, device="cuda")
out = torch.zeros(2, dtype=torch.int64, device="cuda")
for swz, warps in ((1, 1), (1, 4), (1, 8)):
    for rows in (8, 32, 128):
        nbox = (192 * 1024) // (rows * 128) if rows < 256 else 6
        for rep in range(2):
            assert L.tma_probe(g.data_ptr(), 8192, rows, nbox, swz, out.data_ptr(), warps) == 0
        o = out.tolist()
        print(f"warps={warps} swz={swz} rows={rows:4d} boxes={nbox:4d} ({nbox*rows*128//1024} KB): issue {o[0]/1e3:6.2f} us, done {o[1]/1e3:6.2f} us  -> {nbox*rows*128/o[1]:.1f} GB/s")
