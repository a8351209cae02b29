"""Intermittent-NaN hunt: SCC-ResNet-18 training (batch 32) repeated with the
fused dsc forward and / or the one-pass depthwise backward swapped for the
kernel pairs (monkeypatched), counting runs whose losses are not finite; the
caching allocator is filled with NaN before each run."""
import math, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2101_00745_b200 as pkg
from paper_2101_00745_b200 import scc
from paper_2101_00745_b200.train import train_throughput
orig_fwd_t, orig_bwd = scc.dsc_forward_t, scc.dw3x3_backward
def pair_fwd_t(x, dw, db, wts, cfg, stride=1):
    t = scc.dw3x3_forward(x, dw, db, stride)
    return scc.scc_forward(t, wts, cfg), t
def pair_bwd(dy, x, w, stride=1, with_bias=False):
    dx = scc.dw3x3_backward_data(dy, w, x.shape[2:], stride)
    dw, db = scc.dw3x3_backward_weight(dy, x, stride, with_bias)
    return dx, dw, db
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
for mode in sys.argv[2:] or ["both", "pair_fwd", "pair_bwd", "neither"]:
    scc.dsc_forward_t = pair_fwd_t if mode in ("pair_fwd", "neither") else orig_fwd_t
    scc.dw3x3_backward = pair_bwd if mode in ("pair_bwd", "neither") else orig_bwd
    bad = 0
    for i in range(reps):
        # poison the caching allocator: memory a kernel reads without anyone
        # having written it comes back NaN
        junk = torch.full((1 << 28,), float("nan"), device="cuda")
        del junk
        torch.manual_seed(i)
        r = train_throughput("resnet18", batch=32, steps=15, warmup=1)
        if not (math.isfinite(r["loss_first"]) and math.isfinite(r["loss_last"])):
            bad += 1
    print(mode, "non-finite runs:", bad, "of", reps, flush=True)
