"""A/B of the generation-1 band kernel's row-tile width and panel residency,
interleaved in one process (min of 3 rounds): NT=128 (plan default), NT=64
with the per-row-tile resident panel, NT=64 streamed.  Forward, N=32."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
torch.cuda.set_device(0)
SHAPES = [(c, cg, hw) for c in (256, 512, 1024) for cg in (2, 4, 8) for hw in (56, 14)]
def tg(fn, reps=8, it=5):
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        fn(); st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            for _ in range(reps): fn()
        g.replay(); st.synchronize()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(st)
        for _ in range(it): g.replay()
        b.record(st); b.synchronize()
    return a.elapsed_time(b) * 1e3 / (reps * it)
for c, cg, hw in SHAPES:
    xs = [torch.randn(32, c, hw, hw, device="cuda") for _ in range(2 if hw == 56 else 4)]
    cfgs = {}
    for nt in ("128", "64"):
        os.environ["SCC_TC_NT"] = nt
        cfgs[nt] = scc.scc_config_new(c, c, cg, "50%", True)
    os.environ.pop("SCC_TC_NT")
    wts = scc.scc_weights_init(cfgs["128"])
    k = [0]
    def f(cfg):
        def run():
            k[0] += 1
            scc.scc_forward(xs[k[0] % len(xs)], wts, cfg)
        return run
    res = {"nt128": [], "nt64_rt": [], "nt64_stream": []}
    for _ in range(3):
        os.environ.pop("SCC_BAND_NO_RT_PANEL", None)
        res["nt128"].append(tg(f(cfgs["128"])))
        res["nt64_rt"].append(tg(f(cfgs["64"])))
        os.environ["SCC_BAND_NO_RT_PANEL"] = "1"
        res["nt64_stream"].append(tg(f(cfgs["64"])))
    os.environ.pop("SCC_BAND_NO_RT_PANEL", None)
    print(json.dumps({"C": c, "cg": cg, "hw": hw, **{k2: round(min(v), 2) for k2, v in res.items()}}), flush=True)
    del xs
    torch.cuda.empty_cache()
