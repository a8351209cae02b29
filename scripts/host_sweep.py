"""e2e (host-buffer C ABI, pinned memory) of config 1 vs pipeline depth and
graph replay.  One subprocess per setting (env knobs are read per call but
graphs are cached per key).  Usage: python scripts/host_sweep.py"""
import json, os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, json
sys.path.insert(0, ROOT_PLACEHOLDER)
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
for _ in range(5): _lib.check(L.scc_fwd_bwd_host_f32(cfg.handle, n, h, w, *a))
ts = []
for _ in range(5):
    t0 = time.perf_counter()
    for _ in range(20): _lib.check(L.scc_fwd_bwd_host_f32(cfg.handle, n, h, w, *a))
    ts.append((time.perf_counter() - t0) / 20)
t = min(ts)
print(json.dumps({"ms": t * 1e3, "gbs": 4 * n * h * w * (3 * ci + 2 * co) / t / 1e9}))
'''.replace("ROOT_PLACEHOLDER", repr(ROOT))
for graph in (1, 0):
    for k in (1, 2, 3, 4, 6, 8, 16):
        env = dict(os.environ, SCC_HOST_CHUNKS=str(k))
        if not graph:
            env["SCC_HOST_NO_GRAPH"] = "1"
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=300)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-300:]
        print(f"graph={graph} chunks={k}: {line}", flush=True)
