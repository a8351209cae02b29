"""Per-call device time of forward / backward-data on config 1 for each
tensor-core generation (CUDA events over a CUDA graph of 20 calls, inputs
rotated over 8 buffer sets > L2), plus the gen-2 CTA-0 timeline."""
import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib()
shape = [int(v) for v in (sys.argv[1:7] or ["32", "64", "128", "32", "32", "2"])]
N, CI, CO, H, W, CG = shape
cfg = scc.scc_config_new(CI, CO, CG, "50%", True)
R = 8
xs = [torch.randn(N, CI, H, W, device="cuda") for _ in range(R)]
dys = [torch.randn(N, CO, H, W, device="cuda") for _ in range(R)]
ys = [torch.empty(N, CO, H, W, device="cuda") for _ in range(R)]
dxs = [torch.empty(N, CI, H, W, device="cuda") for _ in range(R)]
wts = scc.scc_weights_init(cfg)
def fwd(i, s):
    _lib.check(L.scc_forward_f32(cfg.handle, N, H, W, xs[i].data_ptr(), wts.weight.data_ptr(), wts.bias.data_ptr(), ys[i].data_ptr(), s))
def bwdd(i, s):
    _lib.check(L.scc_backward_data_f32(cfg.handle, N, H, W, dys[i].data_ptr(), wts.weight.data_ptr(), dxs[i].data_ptr(), s))
for path, name in ((_lib.SCC_PATH_TENSOR_STREAMED, "gen1"), (_lib.SCC_PATH_TENSOR, "gen2")):
    cfg.set_path(path)
    for op, f, nbytes in (("fwd", fwd, 4 * N * H * W * (CI + CO)), ("bwd_data", bwdd, 4 * N * H * W * (CI + CO))):
        if path == _lib.SCC_PATH_TENSOR_STREAMED and len(sys.argv) > 7: continue
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for i in range(R): f(i, st.cuda_stream)
            st.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for k in range(20): f(k % R, st.cuda_stream)
            g.replay(); st.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10): g.replay()
            e1.record(st); e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 200
        print(f"{name} {op}: {us:.2f} us/call  {nbytes / us / 1e3:.0f} GB/s", flush=True)
    if path == _lib.SCC_PATH_TENSOR:
        for op, f in (("fwd", fwd), ("bwd_data", bwdd)):
            f(0, torch.cuda.current_stream().cuda_stream); torch.cuda.synchronize()
            buf = (C.c_uint64 * (192 + 2048))()
            n = L.scc_debug_trace(buf, 192 + 2048)
            import statistics
            st = [buf[192 + 2 * i] for i in range(148)]; en = [buf[193 + 2 * i] for i in range(148)]
            t00 = min(st)
            ends = sorted((e - t00) / 1e3 for e in en)
            starts = sorted((x - t00) / 1e3 for x in st)
            print(op, "CTA starts: min %.2f med %.2f max %.2f | epilogue ends: min %.2f med %.2f p90 %.2f max %.2f" % (
                starts[0], statistics.median(starts), starts[-1], ends[0], statistics.median(ends), ends[int(0.9 * len(ends))], ends[-1]))
            t = [buf[128 + i] for i in range(64)]
            t0 = t[0]
            lab = {0: "start", 1: "dep", 2: "tma_c0_last_tile", 3: "panel", 40: "bar_init", 41: "tab_bulk", 42: "tmem_alloc", 43: "sync", 44: "tileiter"}
            for i in range(8): lab[6 + i] = f"mma{i}"; lab[14 + i] = f"epi{i}"; lab[22 + i] = f"cv{i}s"; lab[30 + i] = f"cv{i}e"
            for g in range(4): lab[38 + g] = f"eg{g}ld"; lab[42 + g] = f"eg{g}st"
            print(op, "epi tile1 grp1 [start, ld done, wait_read done, sts done, fence done, tma issued] (us):", [round((t[54 + i] - t0) / 1e3, 3) if t[54 + i] > t0 else 0 for i in range(6)])
            for i in range(8): t[54 + i] = 0
            print(op, "SM clock MHz (CTA0):", (t[48] - t[47]) * 1e3 / max(t[t[49]] - t[0], 1))
            t[47] = t[48] = t[49] = 0
            print(op, " ".join(f"{lab[i]}={(t[i] - t0) / 1e3:.2f}" for i in sorted(lab) if t[i] >= t0 and t[i] - t0 < 1e8))
