import ctypes as C, os, subprocess, torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
so = os.path.join(root, "tests/cuda/_build/tma_chip_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2", "-std=c++17", "-Xcompiler", "-fPIC", "-shared",
                           "-I" + os.path.join(root, "paper_2101_00745_b200/csrc"), "-o", so, os.path.join(root, "tests/cuda/tma_chip_probe.cu")])
L = C.CDLL(so); L.tma_chip.restype = C.c_float
L.tma_chip.argtypes = [C.c_void_p] + [C.c_int] * 5
for cols in (1024, 3136):
    rows = (512 << 20) // (cols * 4)   # 512 MB tensor (> L2)
    g = torch.randn(rows * cols, device="cuda")
    for bw, bh in ((32, 8), (32, 32), (32, 64), (64, 32), (128, 8), (128, 32), (256, 16)):
        if cols % bw: continue
        gbs = L.tma_chip(g.data_ptr(), cols, rows, bw, bh, 64)
        print(f"row stride {cols*4:6d} B: box {bw:3d} px x {bh:3d} rows ({bw*bh*4//1024:3d} KB): {gbs:7.0f} GB/s aggregate")
    del g
