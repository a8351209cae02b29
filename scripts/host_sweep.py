"""e2e (host-buffer C ABI, pinned memory) of config 1 vs the host pipeline's
chunk schedule: SCC_HOST_XCH / SCC_HOST_DYCH give the relative sizes of the
x-pass and dy-pass chunks.  Usage: python scripts/host_sweep.py"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
from paper_2101_00745_b200 import _lib
L = _lib.lib(); torch.cuda.set_device(0)
n, ci, co, h, w = 32, 64, 128, 32, 32
cfg = scc.scc_config_new(ci, co, 2, "50%", True)
pin = lambda *s: torch.randn(*s).pin_memory()
x, dy, wt, b = pin(n, ci, h, w), pin(n, co, h, w), pin(co * 32), pin(co)
y, dx, dw, db = pin(n, co, h, w), pin(n, ci, h, w), pin(co * 32), pin(co)
a = [x.data_ptr(), wt.data_ptr(), b.data_ptr(), dy.data_ptr(), y.data_ptr(), dx.data_ptr(), dw.data_ptr(), db.data_ptr()]
nbytes = 4 * n * h * w * (3 * ci + 2 * co)
def measure():
    for _ in range(5): _lib.check(L.scc_fwd_bwd_host_f32(cfg.handle, n, h, w, *a))
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        for _ in range(20): _lib.check(L.scc_fwd_bwd_host_f32(cfg.handle, n, h, w, *a))
        ts.append((time.perf_counter() - t0) / 20)
    ts.sort()
    return ts[0] * 1e3, ts[3] * 1e3
schedules = [("", "")] + [(xs, ds) for xs in ("1", "1,1", "1,3", "1,2,4", "1,3,8", "1,1,2,4", "1,2,4,8")
                          for ds in ("1", "1,1,1", "2,1,1", "4,2,1,1", "3,2,1", "6,4,2,1,1", "8,4,2,1,1")]
res = []
for xs, ds in schedules:
    for k, v in (("SCC_HOST_XCH", xs), ("SCC_HOST_DYCH", ds)):
        if v: os.environ[k] = v
        else: os.environ.pop(k, None)
    best, med = measure()
    res.append((best, xs, ds))
    print(json.dumps({"xch": xs or "default", "dych": ds or "default", "ms_best": round(best, 4), "ms_median": round(med, 4),
                      "gbs": round(nbytes / best / 1e6, 1)}), flush=True)
res.sort()
print("best:", res[:5])
