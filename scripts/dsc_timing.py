"""Fused dsc_block forward (scc_dsc_forward_f32) vs the unfused pair (stock
depthwise conv + the SCC forward kernels) at the SCC-ResNet-18 CIFAR layer
shapes (batch 128); device us per call, CUDA graphs of 10 calls."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2101_00745_b200 as scc
torch.cuda.set_device(0)
N = 128
SHAPES = [(64, 64, 32, 1), (64, 128, 32, 2), (128, 128, 16, 1), (128, 256, 16, 2),
          (256, 256, 8, 1), (256, 512, 8, 2), (512, 512, 4, 1)]
def t_graph(fn, reps=10, it=5):
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
rows = []
for ci, co, hw, s in SHAPES:
    cfg = scc.scc_config_new(ci, co, 2, "50%", False)
    x = torch.randn(N, ci, hw, hw, device="cuda")
    dw = torch.randn(ci, 1, 3, 3, device="cuda") / 3
    wts = scc.scc_weights_init(cfg)
    fused = lambda: scc.dsc_forward(x, dw, None, wts, cfg, s)
    unfused = lambda: scc.scc_forward(torch.nn.functional.conv2d(x, dw, None, s, 1, 1, ci), wts, cfg)
    t = torch.nn.functional.conv2d(x, dw, None, s, 1, 1, ci)
    dwonly = lambda: torch.nn.functional.conv2d(x, dw, None, s, 1, 1, ci)
    tc = lambda: scc.scc_forward(t, wts, cfg)
    r = {"c_in": ci, "c_out": co, "hw": hw, "stride": s, "fused_us": round(t_graph(fused), 2),
         "unfused_us": round(t_graph(unfused), 2), "dw_us": round(t_graph(dwonly), 2),
         "scc_tc_us": round(t_graph(tc), 2)}
    gy = torch.randn_like(t)
    r["dw_ours_us"] = round(t_graph(lambda: scc.dw3x3_forward(x, dw, None, s)), 2)
    # the training forward: y and t (the SCC backward's input) from one call
    r["fused_t_us"] = round(t_graph(lambda: scc.dsc_forward_t(x, dw, None, wts, cfg, s)), 2)
    r["pair_ours_us"] = round(t_graph(lambda: scc.scc_forward(scc.dw3x3_forward(x, dw, None, s), wts, cfg)), 2)
    r["dw_bwd_data_ours_us"] = round(t_graph(lambda: scc.dw3x3_backward_data(gy, dw, (hw, hw), s)), 2)
    r["dw_bwd_weight_ours_us"] = round(t_graph(lambda: scc.dw3x3_backward_weight(gy, x, s)), 2)
    r["dw_bwd_data_torch_us"] = round(t_graph(lambda: torch.nn.grad.conv2d_input(x.shape, dw, gy, s, 1, 1, ci)), 2)
    r["dw_bwd_ours_us"] = round(t_graph(lambda: scc.dw3x3_backward(gy, x, dw, s)), 2)
    r["dw_bwd_weight_torch_us"] = round(t_graph(lambda: torch.nn.grad.conv2d_weight(x, dw.shape, gy, s, 1, 1, ci)), 2)
    cfg.set_path(1)  # SCC_PATH_CUDA_CORE
    r["scc_cc_us"] = round(t_graph(tc), 2)
    rows.append(r); print(json.dumps(r), flush=True)
