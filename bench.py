#!/usr/bin/env python
"""Benchmark of the SCC hot path (BASELINE.json metric: SCC fwd+bwd GB/s, %
of the HBM roofline).

Workload (BASELINE.json configs[0], the layer shape the metric is quoted on):
one SCC layer, fp32, N=32 per GPU, C_in=64 -> C_out=128, H=W=32, cg=2,
co=50%.  One step = forward + backward-data + backward-weight (+ the NCCL
all-reduce of dW/db across ranks when N>1: the data-parallel exchange of
north_star).  Algorithmic bytes per step = 4*N*H*W*(3*C_in + 2*C_out)
(weights are negligible).  Inputs rotate over enough buffer sets
to exceed 3x L2, so every step streams from HBM.

  python bench.py [--gpus N --steps K --warmup W]           # our kernels
  python bench.py --impl reference [...]                     # reference CPU path
Under torchrun (N>1) every rank runs its own shard (weak scaling) and rank 0
prints one JSON line.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (c_in, c_out, cg, co, n, h, w)
    "c1": (64, 128, 2, "50%", 32, 32, 32),
}
for _c in (256, 512, 1024):
    for _cg in (2, 4, 8):
        for _co in (25, 50, 75):
            for _hw in (56, 14):
                WORKLOADS[f"sweep_C{_c}_cg{_cg}_co{_co}_{_hw}"] = (_c, _c, _cg, f"{_co}%", 32, _hw, _hw)

METRIC = "SCC fwd+bwd GB/s (% HBM roofline)"


def workload_desc(name):
    """config.workload, identical in both arms (the driver compares them)."""
    ci, co, cg, ov, n, h, w = WORKLOADS[name]
    return (f"{name}: SCC layer fwd+bwd fp32 NCHW, N={n}/GPU C_in={ci} C_out={co} "
            f"H=W={h} cg={cg} co={ov}")


def algo_bytes(ci, co, n, h, w):
    """Compulsory fp32 bytes of fwd + bwd."""
    p = n * h * w
    return {
        "step": 4 * p * (3 * ci + 2 * co),
        "forward": 4 * p * (ci + co),
        "backward_data": 4 * p * (co + ci),
        "backward_weight": 4 * p * (co + ci),
        # scc_backward_f32 as the step runs it: dy read once (fused kernel) or
        # dx / dW concurrently; compulsory bytes = dy + x read, dx written
        "backward": 4 * p * (2 * ci + co),
    }


def algo_flops(ci, co, gw, n, h, w):
    return 2 * n * h * w * co * gw  # per pass (cost.cpp:91 MACs x 2)


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1590.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the GPU is busy."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []
        self._t = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self._t:
            self._t.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


# ---------------------------------------------------------------------------
# reference CPU arm


def reference_problem(workload, n_override=None):
    from oracle import load_port, load_ref
    ci, co, cg, ov, n, h, w = WORKLOADS[workload]
    if n_override:
        n = n_override
    ref = load_ref()
    kind = "reference"
    if ref is None:
        ref, kind = load_port(), "port"
    if kind == "reference":
        ref.set_num_threads(os.cpu_count() or 1)
        cores = ref.num_threads()
        cfg = ref.config(ci, co, cg, ov, True)
    else:
        cores = 1
        cfg = ref.config(ci, co, cg, ("ratio", float(ov[:-1]) / 100), True)
    rng = np.random.default_rng(0)
    x = rng.standard_normal((n, ci, h, w)).astype(np.float32)
    wt = rng.uniform(-1, 1, co * cfg.group_width).astype(np.float32) * np.float32(
        np.sqrt(1.0 / cfg.group_width))
    b = rng.uniform(-0.5, 0.5, co).astype(np.float32)
    dy = rng.standard_normal((n, co, h, w)).astype(np.float32)
    if kind == "reference":
        prob = ref.problem(cfg, x, wt, b, dy)
        step = prob.step
    else:
        def step():
            ref.forward(cfg, x, wt, b)
            ref.backward_input(cfg, dy, wt)
            ref.backward_params(cfg, dy, x)
            return 0.0
    return step, kind, cores, n, (ci, co, h, w)


def time_reference(workload, steps, warmup, budget_s=None, n_override=None):
    step, kind, cores, n, (ci, co, h, w) = reference_problem(workload, n_override)
    for _ in range(max(warmup, 1)):
        step()
    times = []
    t_all = time.perf_counter()
    for i in range(steps):
        t0 = time.perf_counter()
        step()
        times.append(time.perf_counter() - t0)
        if budget_s is not None and time.perf_counter() - t_all > budget_s and i >= 1:
            break
    mean = sum(times) / len(times)
    gbs = algo_bytes(ci, co, n, h, w)["step"] / mean / 1e9
    return {"value": gbs, "unit": "GB/s", "cores": cores, "kind": kind,
            "sample": (f"{len(times)} fwd+bwd steps of {workload} at N={n} "
                       f"(fp64 reference arithmetic on fp32-valued inputs), mean {mean*1e3:.1f} ms/step"),
            "ms_per_step": mean * 1e3, "steps": len(times)}


def run_reference_arm(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    r = time_reference(args.workload, args.steps, args.warmup)
    ci, co, cg, ov, n, h, w = WORKLOADS[args.workload]
    line = {
        "impl": "reference",
        "metric": METRIC, "value": round(r["value"], 4), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": r["steps"], "warmup": args.warmup,
        "ms_per_step": round(r["ms_per_step"], 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args.workload),
                   "device": "host CPU", "parallelism": "host threads"},
        "cpu_baseline": {"value": round(r["value"], 4), "unit": "GB/s", "cores": r["cores"],
                         "kind": r["kind"], "sample": r["sample"]},
        "e2e": {"value": round(r["value"], 4), "unit": "GB/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm


def measure_traffic(workload, timeout=240):
    """roofline.traffic, measured in this run: scripts/traffic_probe.py under
    ncu (dram__bytes_read + dram__bytes_write of the step's kernels, plus the
    dirty lines they leave in L2, evicted by a read-only flush that follows).
    A separate process: no number here is timed under the profiler."""
    import tempfile
    csv_path = os.path.join(tempfile.mkdtemp(prefix="scc_traffic_"), "t.csv")
    cmd = ["ncu", "--metrics", "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum",
           "--clock-control", "none", "--cache-control", "none", "--print-units", "base", "--csv", "--log-file", csv_path,
           sys.executable, os.path.join(ROOT, "scripts", "traffic_probe.py"), "--workload", workload]
    try:
        subprocess.run(cmd, stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL, timeout=timeout,
                       env=dict(os.environ, CUDA_VISIBLE_DEVICES=os.environ.get("CUDA_VISIBLE_DEVICES", "0")))
        sys.path.insert(0, os.path.join(ROOT, "scripts"))
        from traffic_probe import parse
        d = parse(csv_path)
        d["method"] = ("ncu dram__bytes_read.sum + dram__bytes_write.sum of the phase's kernels "
                       "+ dram__bytes_write.sum of the read-only L2 flush that follows (scripts/traffic_probe.py)")
        return d
    except Exception as ex:  # reported, never required
        return {"error": f"traffic pass failed: {str(ex)[:160]}"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2101_00745_b200 as scc
    from paper_2101_00745_b200 import _lib
    from paper_2101_00745_b200.dist import allreduce_grads

    ws, rank, local = dist_env()
    if ws > 1:
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    ci, co, cg, ov, n, h, w = WORKLOADS[args.workload]
    cfg = scc.scc_config_new(ci, co, cg, ov, True)
    if args.path:
        cfg.set_path({"cc": _lib.SCC_PATH_CUDA_CORE, "tc": _lib.SCC_PATH_TENSOR}[args.path])
    gw = cfg.group_width
    hbm_peak, _, peak_kind = peaks()
    nbytes = algo_bytes(ci, co, n, h, w)

    # Rotating buffer sets > 3x L2 so each step streams from HBM.
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    per_set = 4 * n * h * w * (2 * ci + 2 * co)
    nsets = max(2, min(64, -(-3 * l2 // per_set)))
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    sets = []
    for _ in range(nsets):
        x = torch.randn(n, ci, h, w, device=dev, generator=gen)
        dy = torch.randn(n, co, h, w, device=dev, generator=gen)
        y = torch.empty(n, co, h, w, device=dev)
        dx = torch.empty(n, ci, h, w, device=dev)
        sets.append((x, dy, y, dx))
    bound = (1.0 / gw) ** 0.5
    weight = (torch.rand(co * gw, device=dev, generator=gen) * 2 - 1) * bound
    bias = torch.rand(co, device=dev, generator=gen) - 0.5
    dw = torch.empty(co * gw, device=dev)
    db = torch.empty(co, device=dev)
    grads = torch.empty(co * gw + co, device=dev)
    wsb = cfg.workspace_bytes(n, h, w)
    wsbuf = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    L = _lib.lib()
    h_ = cfg.handle
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def fwd(i):
        x, dy, y, dx = sets[i % nsets]
        _lib.check(L.scc_forward_f32(h_, n, h, w, x.data_ptr(), weight.data_ptr(),
                                     bias.data_ptr(), y.data_ptr(), sp))

    def bwd(i):
        x, dy, y, dx = sets[i % nsets]
        _lib.check(L.scc_backward_f32(h_, n, h, w, dy.data_ptr(), x.data_ptr(), weight.data_ptr(),
                                      dx.data_ptr(), grads.data_ptr(), grads.data_ptr() + 4 * co * gw,
                                      wsbuf.data_ptr(), wsb, sp))

    def bwd_data(i):
        x, dy, y, dx = sets[i % nsets]
        _lib.check(L.scc_backward_data_f32(h_, n, h, w, dy.data_ptr(), weight.data_ptr(),
                                           dx.data_ptr(), sp))

    def bwd_weight(i):
        x, dy, y, dx = sets[i % nsets]
        _lib.check(L.scc_backward_weight_f32(h_, n, h, w, dy.data_ptr(), x.data_ptr(),
                                             dw.data_ptr(), db.data_ptr(), wsbuf.data_ptr(), wsb, sp))

    def step(i):
        fwd(i)
        bwd(i)
        if ws > 1:
            # data-parallel exchange of dW|db (north_star): one flat bucket,
            # reduced in place (dist.py, the same call train.py makes)
            allreduce_grads([grads], average=True)

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # CUDA graphs: one graph holds one full rotation of `nsets` consecutive
    # steps (plus one graph per single step for a remainder), so the device
    # time is not bounded by per-launch host overhead.  Warm up on the capture
    # stream first (plan tables, per-stream scratch, fork/join streams, NCCL).
    graphs = None
    if not args.no_graph:
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            sp_saved = sp
            sp = cap.cuda_stream
            for i in range(nsets):
                step(i)
            torch.cuda.synchronize()
            g_all = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g_all, stream=cap):
                for i in range(nsets):
                    step(i)
            graphs = []
            for i in range(nsets):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step(i)
                graphs.append(g)
            sp = sp_saved
        torch.cuda.synchronize()

    def run_step(i):
        if graphs is not None:
            graphs[i % nsets].replay()
        else:
            step(i)

    def run_steps(k):
        # exactly k steps: whole rotations through the multi-step graph, the
        # remainder through single-step graphs
        if graphs is None:
            for i in range(k):
                step(i)
            return
        for _ in range(k // nsets):
            g_all.replay()
        for i in range(k % nsets):
            graphs[i].replay()

    sampler = ClockSampler(dev.index if ws == 1 else local)
    sampler.start()
    for i in range(max(args.warmup, 3)):
        run_step(i)
    barrier()
    # keep the GPU busy ~1 s before timing so the clock record is under load
    t_end = time.perf_counter() + 1.0
    i = 0
    while time.perf_counter() < t_end:
        for _ in range(20):
            run_step(i)
            i += 1
        torch.cuda.synchronize()
    barrier()

    # kernels per step, counted on an eager step (graph replays do not pass
    # through the host library)
    c0 = L.scc_launch_count()
    step(0)
    torch.cuda.synchronize()
    per_step_launches = L.scc_launch_count() - c0

    # ---- timed region (value) ----
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    barrier()
    e0.record(stream)
    run_steps(args.steps)
    e1.record(stream)
    barrier()
    launches = per_step_launches * args.steps
    ms = e0.elapsed_time(e1)
    if ws > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    clocks = sampler.stop()
    ms_step = ms / args.steps
    value = nbytes["step"] * ws / (ms_step * 1e-3) / 1e9

    # ---- per-kernel timing (roofline of the dominant kernel) ----
    # The step launches forward + scc_backward_f32; the dominant of those two
    # is the roofline kernel.  backward-data / backward-weight alone are
    # reported for reference (kernel_ms) but are not what the step runs.
    # Each part is replayed from a CUDA graph of 16 calls (rotating over the
    # buffer sets, like the step), so host launch overhead is not timed.
    parts = {"forward": fwd, "backward": bwd, "backward_data": bwd_data, "backward_weight": bwd_weight}
    kms = {}
    reps = max(args.steps // 16, 4)
    pstream = cap if graphs is not None else stream
    sp_saved = sp
    sp = pstream.cuda_stream
    with torch.cuda.stream(pstream):
        for name, fn in parts.items():
            for i in range(3):
                fn(i)
            torch.cuda.synchronize()
            pg = None
            if graphs is not None:
                pg = torch.cuda.CUDAGraph()
                with torch.cuda.graph(pg, stream=pstream):
                    for i in range(16):
                        fn(i)
                pg.replay()
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(pstream)
            for r in range(reps):
                if pg is None:
                    for i in range(16):
                        fn(i)
                else:
                    pg.replay()
            b.record(pstream)
            b.synchronize()
            kms[name] = a.elapsed_time(b) / (16 * reps)
    sp = sp_saved
    dominant = max(("forward", "backward"), key=kms.get)
    achieved = nbytes[dominant] / (kms[dominant] * 1e-3) / 1e9
    traffic, traffic_detail = None, None
    if rank == 0 and ws == 1 and not args.no_traffic:
        traffic_detail = measure_traffic(args.workload)
        if traffic_detail and dominant in traffic_detail:
            traffic = int(traffic_detail[dominant]["total"])
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm_peak, "unit": "GB/s",
                "frac": round(achieved / hbm_peak, 4), "traffic": traffic,
                "traffic_detail": traffic_detail,
                "kernel": dominant, "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": nbytes[dominant],
                "kernel_ms": {k: round(v, 5) for k, v in kms.items()},
                "step_frac": round(value / ws / hbm_peak, 4)}

    # ---- end to end through the host-buffer C ABI (pinned host memory) ----
    e2e = None
    if not args.no_e2e:
        xh = torch.randn(n, ci, h, w).pin_memory()
        dyh = torch.randn(n, co, h, w).pin_memory()
        wh = weight.cpu().pin_memory()
        bh = bias.cpu().pin_memory()
        yh = torch.empty(n, co, h, w).pin_memory()
        dxh = torch.empty(n, ci, h, w).pin_memory()
        dwh = torch.empty(co * gw).pin_memory()
        dbh = torch.empty(co).pin_memory()
        args_h = [xh.data_ptr(), wh.data_ptr(), bh.data_ptr(), dyh.data_ptr(), yh.data_ptr(),
                  dxh.data_ptr(), dwh.data_ptr(), dbh.data_ptr()]
        for _ in range(3):
            _lib.check(L.scc_fwd_bwd_host_f32(h_, n, h, w, *args_h))
        barrier()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            _lib.check(L.scc_fwd_bwd_host_f32(h_, n, h, w, *args_h))
        dt = (time.perf_counter() - t0) / args.steps
        if ws > 1:
            t = torch.tensor([dt], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t.item())
        h2d = 4 * (xh.numel() + wh.numel() + bh.numel() + dyh.numel())
        d2h = 4 * (yh.numel() + dxh.numel() + dwh.numel() + dbh.numel())
        e2e = {"value": round(nbytes["step"] * ws / dt / 1e9, 3), "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "ms_per_step": round(dt * 1e3, 4),
               "api": "scc_fwd_bwd_host_f32 (include/scc_b200.h)"}

    # ---- BASELINE configs C2-C4: SCC-VGG16 / SCC-ResNet-18 / SCC-ResNet-50 images/sec ----
    models = None
    if not args.no_models:
        from paper_2101_00745_b200.train import train_throughput
        models = {}
        runs = {"resnet18": dict(batch=128, steps=20, warmup=5),            # C3 (CIFAR shape)
                "vgg16": dict(batch=128, steps=20, warmup=5),               # C2 (CIFAR shape)
                "resnet50": dict(batch=256, steps=8, warmup=3, image=224,   # C4 (ImageNet shape;
                                 num_classes=1000),                         # paper rule, 12.87 M)
                "resnet50_all": dict(batch=256, steps=8, warmup=3, image=224,  # every 1x1 -> SCC
                                     num_classes=1000)}
        for name, kw in runs.items():
            try:
                models[name] = train_throughput(name, **kw)
            except Exception as ex:  # reported, never required for the headline
                models[name] = {"error": str(ex)[:200]}

    # ---- the paper's Base vs Opt on this GPU: one layer step through the
    # stock-operator compositions (reference.cpp:335-490) vs the SCC kernels
    compositions = None
    if rank == 0 and ws == 1 and not args.no_compositions and args.workload == "c1":
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            from compose_bench import SHAPES, run_shape
            compositions = run_shape("c1", *SHAPES["c1"])
        except Exception as ex:  # reported, never required for the headline
            compositions = {"error": str(ex)[:200]}

    # ---- BASELINE config C5 (the design-space sweep), a representative subset
    # timed in this run: cg=4, co=50 % at every (C, H x W) -- the full 54-shape
    # sweep is scripts/sweep.py (profiles/*_sweep_c5.json)
    c5 = None
    if rank == 0 and ws == 1 and not args.no_c5 and args.workload == "c1":
        try:
            sys.path.insert(0, os.path.join(ROOT, "scripts"))
            import sweep as c5sweep
            hbm_peak, _ = c5sweep.peaks()
            rows = []
            st5 = torch.cuda.Stream()
            for hw in (56, 14):
                for c in (256, 512, 1024):
                    r = c5sweep.run_shape(c, 4, 50, hw, 32, _lib.lib(), st5)
                    r["hbm_frac_step"] = round(r["gbs"]["step"] / hbm_peak, 4)
                    rows.append({k: r[k] for k in ("C", "hw", "cg", "co", "gw", "us", "gbs", "hbm_frac_step")})
                    torch.cuda.empty_cache()
            fr = sorted(r["hbm_frac_step"] for r in rows)
            c5 = {"subset": "C in {256,512,1024} x H=W in {56,14}, cg=4, co=50%, N=32; fwd / bwd / step "
                            "= forward, scc_backward_f32, both (CUDA graphs of 8 calls, inputs > 3x L2)",
                  "rows": rows, "hbm_frac_step_median": round((fr[2] + fr[3]) / 2, 4),
                  "hbm_frac_step_min": fr[0], "hbm_frac_step_max": fr[-1]}
        except Exception as ex:  # reported, never required for the headline
            c5 = {"error": str(ex)[:200]}

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        try:
            r = time_reference(args.workload, steps=20, warmup=1, budget_s=args.cpu_budget)
            cpu = {k: r[k] for k in ("value", "unit", "cores", "kind", "sample")}
            cpu["value"] = round(cpu["value"], 4)
        except Exception as ex:  # baseline is reported, never required
            cpu = {"value": None, "unit": "GB/s", "cores": 0, "kind": "unavailable",
                   "sample": f"reference CPU path failed: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 5),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(args.workload), "gw": gw, "shift": cfg.shift,
                       "global_batch": n * ws, "parallelism": f"dp{ws}",
                       "l2": f"inputs rotate over {nsets} buffer sets "
                             f"({nsets * per_set / 2**20:.0f} MiB > 3x L2 {l2 / 2**20:.0f} MiB)",
                       "path": {1: "cuda_core", 2: "tensor"}.get(cfg.path_for(n, h, w), "?"),
                       "bytes_per_step_per_gpu": nbytes["step"],
                       "collective": "NCCL all_reduce(dW,db) per step" if ws > 1 else "none",
                       "launch": "eager" if graphs is None else f"CUDA graphs of {nsets} steps"},
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "models": models,
            "compositions": compositions,
            "c5": c5,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c1", choices=sorted(WORKLOADS))
    ap.add_argument("--path", default=None, choices=[None, "cc", "tc"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch each step eagerly")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-models", action="store_true", help="skip the SCC-ResNet-18/VGG16 images/sec")
    ap.add_argument("--no-compositions", action="store_true",
                    help="skip the stock-operator (paper 'Base') composition timings")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 sweep subset")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--no-traffic", action="store_true", help="skip the ncu DRAM-traffic pass")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference_arm(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
