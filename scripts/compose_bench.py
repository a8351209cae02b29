"""The paper's Base vs Opt comparison on the B200: one training step of an SCC
layer (forward + dx, dW, db) through the composition routes built from stock
PyTorch operators (paper_2101_00745_b200/compose.py = reference.cpp:335-490:
channel stack / conv stack, with and without the channel-cyclic sharing)
against the SCC kernels (scc_forward_f32 + scc_backward_f32).  fp32, TF32
off; every variant is replayed from a CUDA graph over 4 rotating input sets;
CUDA events on the replay stream.

Usage: python scripts/compose_bench.py [--out FILE] [--shapes c1|all]"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

SHAPES = {
    "c1": (32, 64, 128, 32, 32, 2, "50%"),
    "C256_56_cg2": (32, 256, 256, 56, 56, 2, "50%"),
    "C256_14_cg8": (32, 256, 256, 14, 14, 8, "50%"),
    "C512_14_cg4": (32, 512, 512, 14, 14, 4, "50%"),
}


def time_graph(fn, sets, reps=10):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        for i in range(len(sets)):
            fn(sets[i])
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for s in sets:
                fn(s)
        g.replay()
        st.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(reps):
            g.replay()
        b.record(st)
        b.synchronize()
    return a.elapsed_time(b) / (reps * len(sets))


def run_shape(name, n, ci, co, h, w, cg, ov, max_stack_gb=40.0):
    import paper_2101_00745_b200 as scc
    from paper_2101_00745_b200 import _lib, compose
    torch.backends.cudnn.allow_tf32 = False
    torch.backends.cuda.matmul.allow_tf32 = False
    torch.backends.cudnn.benchmark = True
    cfg = scc.scc_config_new(ci, co, cg, ov, True)
    gw = cfg.group_width
    wts = scc.scc_weights_init(cfg)
    L = _lib.lib()
    nsets = 4
    sets = []
    for _ in range(nsets):
        sets.append(dict(x=torch.randn(n, ci, h, w, device="cuda"), dy=torch.randn(n, co, h, w, device="cuda"),
                         y=torch.empty(n, co, h, w, device="cuda"), dx=torch.empty(n, ci, h, w, device="cuda")))
    grads = torch.empty(co * gw + co, device="cuda")
    wsb = cfg.workspace_bytes(n, h, w)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device="cuda")
    bytes_step = 4 * n * h * w * (3 * ci + 2 * co)
    res = {"shape": name, "n": n, "c_in": ci, "c_out": co, "hw": h, "cg": cg, "co": ov,
           "stacked_gb": round(4 * n * co * gw * h * w / 1e9, 2), "ms": {}}

    def ours(s):
        sp = torch.cuda.current_stream().cuda_stream
        _lib.check(L.scc_forward_f32(cfg.handle, n, h, w, s["x"].data_ptr(), wts.weight.data_ptr(),
                                     wts.bias.data_ptr(), s["y"].data_ptr(), sp))
        _lib.check(L.scc_backward_f32(cfg.handle, n, h, w, s["dy"].data_ptr(), s["x"].data_ptr(),
                                      wts.weight.data_ptr(), s["dx"].data_ptr(), grads.data_ptr(),
                                      grads.data_ptr() + 4 * co * gw, ws.data_ptr(), wsb, sp))
    res["ms"]["scc_kernels"] = time_graph(ours, sets)
    for route in ("channel", "conv"):
        for use_cc in (False, True):
            key = f"{route}_stack{'_cc' if use_cc else ''}"
            if route == "channel" and res["stacked_gb"] > max_stack_gb:
                res["ms"][key] = None
                continue
            def base(s, route=route, use_cc=use_cc):
                compose.compose_backward(route, use_cc, s["dy"], s["x"], wts.weight, wts.bias, cfg)
            try:
                res["ms"][key] = time_graph(base, sets, reps=3 if route == "conv" else 10)
            except torch.cuda.OutOfMemoryError:
                res["ms"][key] = None
            torch.cuda.empty_cache()
    ms = res["ms"]
    res["gbs_scc"] = round(bytes_step / (ms["scc_kernels"] * 1e-3) / 1e9, 1)
    res["speedup_vs"] = {k: (round(v / ms["scc_kernels"], 2) if v else None) for k, v in ms.items() if k != "scc_kernels"}
    for k in ms:
        ms[k] = None if ms[k] is None else round(ms[k], 4)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--shapes", default="all")
    a = ap.parse_args()
    names = ["c1"] if a.shapes == "c1" else list(SHAPES)
    rows = []
    for nm in names:
        r = run_shape(nm, *SHAPES[nm])
        rows.append(r)
        print(json.dumps(r), flush=True)
    if a.out:
        with open(a.out, "w") as f:
            json.dump(rows, f, indent=1)


if __name__ == "__main__":
    main()
