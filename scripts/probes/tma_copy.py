"""Forward-shaped I/O with no compute (tests/cuda/tma_copy_probe.cu): x [32][64][1024]
read once, written twice into y [32][128][1024]; us per launch (back to back)."""
import ctypes as C, os
import torch
root = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
L = C.CDLL(os.path.join(root, "tests/cuda/_build/tma_copy_probe.so")); L.tma_copy.restype = C.c_float
L.tma_copy.argtypes = [C.c_void_p, C.c_void_p] + [C.c_int] * 5
x = torch.randn(32, 64, 1024, device="cuda"); y = torch.empty(32, 128, 1024, device="cuda")
nb = 4 * 32 * 1024 * (64 + 128)
for depth in (2, 4, 8, 12):
    for grid in (148, 296):
        us = L.tma_copy(x.data_ptr(), y.data_ptr(), 32, 64, 1024, depth, grid)
        print(f"depth {depth:2d} grid {grid}: {us:.2f} us  {nb / us / 1e3:.0f} GB/s", flush=True)
