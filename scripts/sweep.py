"""BASELINE config C5: the SCC layer design-space sweep.

Ci = Co = C in {256, 512, 1024}, H = W in {56, 14}, cg in {2, 4, 8},
co in {25, 50, 75}%, N = 32.  For every shape: device time per call of the
forward, the backward (scc_backward_f32) and forward+backward, each as CUDA
graphs of 8 calls, inputs rotated over enough buffer sets to exceed 3x L2
(126 MB).  GB/s = compulsory bytes (fwd+bwd = 4*N*P*(3Ci+2Co)) / time; frac =
GB/s / the measured HBM copy peak (MEASURED_PEAKS.json); tensor-pipe share of
the 3xTF32 work is reported against bf16 dense / 2 / 3.

Usage: python scripts/sweep.py [--co 50] [--out profiles/r01_sweep.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2101_00745_b200 as scc  # noqa: E402
from paper_2101_00745_b200 import _lib  # noqa: E402

L2 = 126 << 20
PARTS = False


def peaks():
    try:
        d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
        return float(d["hbm_gbs"]), float(d["bf16_tflops"])
    except Exception:
        return 6650.0, 1590.0


def time_graph(fn, sets, st, reps=8, iters=5):
    with torch.cuda.stream(st):
        for i in range(sets):
            fn(i, st.cuda_stream)
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for k in range(reps):
                fn(k % sets, st.cuda_stream)
        g.replay()
        st.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            g.replay()
        e1.record(st)
        e1.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (reps * iters)  # us per call


def run_shape(c, cg, co, hw, n, L, st):
    cfg = scc.scc_config_new(c, c, cg, f"{co}%", True)
    gw = cfg.group_width
    P = hw * hw
    set_bytes = 4 * n * P * (c + c) * 2  # x, dx, y, dy
    sets = max(1, min(8, -(-3 * L2 // set_bytes)))
    xs = [torch.randn(n, c, hw, hw, device="cuda") for _ in range(sets)]
    dys = [torch.randn(n, c, hw, hw, device="cuda") for _ in range(sets)]
    ys = [torch.empty(n, c, hw, hw, device="cuda") for _ in range(sets)]
    dxs = [torch.empty(n, c, hw, hw, device="cuda") for _ in range(sets)]
    wts = scc.scc_weights_init(cfg)
    ws = torch.empty(max(1, cfg.workspace_bytes(n, hw, hw)), dtype=torch.uint8, device="cuda")
    gb = torch.empty(c * gw + c, device="cuda")
    wp, bp = wts.weight.data_ptr(), wts.bias.data_ptr()

    def fwd(i, s):
        _lib.check(L.scc_forward_f32(cfg.handle, n, hw, hw, xs[i].data_ptr(), wp, bp, ys[i].data_ptr(), s))

    def bwd(i, s):
        _lib.check(L.scc_backward_f32(cfg.handle, n, hw, hw, dys[i].data_ptr(), xs[i].data_ptr(), wp,
                                      dxs[i].data_ptr(), gb.data_ptr(), gb.data_ptr() + 4 * c * gw,
                                      ws.data_ptr(), ws.numel(), s))

    def both(i, s):
        fwd(i, s)
        bwd(i, s)

    def bdata(i, s):
        _lib.check(L.scc_backward_data_f32(cfg.handle, n, hw, hw, dys[i].data_ptr(), wp, dxs[i].data_ptr(), s))

    def bweight(i, s):
        _lib.check(L.scc_backward_weight_f32(cfg.handle, n, hw, hw, dys[i].data_ptr(), xs[i].data_ptr(),
                                             gb.data_ptr(), gb.data_ptr() + 4 * c * gw, ws.data_ptr(), ws.numel(), s))

    t_f = time_graph(fwd, sets, st)
    t_b = time_graph(bwd, sets, st)
    t_s = time_graph(both, sets, st)
    parts = {}
    if PARTS:
        parts = {"bwd_data": round(time_graph(bdata, sets, st), 2), "bwd_weight": round(time_graph(bweight, sets, st), 2)}
    path = {0: "auto", 1: "cuda_core", 2: "tensor", 3: "tensor_streamed"}.get(cfg.path_for(n, hw, hw), "?") \
        if hasattr(cfg, "path_for") else None
    del xs, dys, ys, dxs
    byt = {"fwd": 4 * n * P * 2 * c, "bwd": 4 * n * P * 3 * c, "step": 4 * n * P * 5 * c}
    flops = 6 * n * P * c * gw
    return {"C": c, "cg": cg, "co": co, "hw": hw, "n": n, "gw": gw, "shift": cfg.shift, "path": path,
            "us": {"fwd": round(t_f, 2), "bwd": round(t_b, 2), "step": round(t_s, 2), **parts},
            "gbs": {k: round(byt[k] / (t * 1e3), 1) for k, t in (("fwd", t_f), ("bwd", t_b), ("step", t_s))},
            "tflops_step": round(flops / (t_s * 1e6), 1), "bytes_step": byt["step"]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--co", type=int, nargs="*", default=[25, 50, 75])
    ap.add_argument("--C", type=int, nargs="*", default=[256, 512, 1024])
    ap.add_argument("--cg", type=int, nargs="*", default=[2, 4, 8])
    ap.add_argument("--hw", type=int, nargs="*", default=[56, 14])
    ap.add_argument("--n", type=int, default=32)
    ap.add_argument("--out", default=None)
    ap.add_argument("--parts", action="store_true", help="also time backward-data / backward-weight alone")
    a = ap.parse_args()
    global PARTS
    PARTS = a.parts
    torch.cuda.set_device(0)
    L = _lib.lib()
    hbm, bf16 = peaks()
    tc_peak = bf16 / 2 / 3  # 3xTF32 on the tensor pipe
    st = torch.cuda.Stream()
    rows = []
    for c in a.C:
        for hw in a.hw:
            for cg in a.cg:
                for co in a.co:
                    r = run_shape(c, cg, co, hw, a.n, L, st)
                    r["hbm_frac_step"] = round(r["gbs"]["step"] / hbm, 4)
                    r["tc_frac_step"] = round(r["tflops_step"] / tc_peak, 4)
                    rows.append(r)
                    print(json.dumps(r), flush=True)
                    torch.cuda.empty_cache()
    fr = sorted(r["hbm_frac_step"] for r in rows)
    summary = {"shapes": len(rows), "hbm_peak_gbs": hbm, "tf32x3_peak_tflops": round(tc_peak, 1),
               "hbm_frac_step_min": fr[0], "hbm_frac_step_median": fr[len(fr) // 2], "hbm_frac_step_max": fr[-1]}
    print(json.dumps({"summary": summary}), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump({"summary": summary, "rows": rows}, f, indent=1)


if __name__ == "__main__":
    main()
