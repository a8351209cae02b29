"""Copies-only timeline of the host pipeline's schedule at config 1 (x chunks,
then dy chunks on the H2D stream; y chunks after their x chunk, dx chunks
after their dy chunk on the D2H stream).  Prints each copy's start / end (us)
and the PCIe rates, for chunk counts 1..8."""
import sys, torch
N, CI, CO, P = 32, 64, 128, 1024
pin = lambda *s: torch.empty(*s).pin_memory()
hx, hdy, hy, hdx = pin(N, CI * P), pin(N, CO * P), pin(N, CO * P), pin(N, CI * P)
dx_, ddy, dy_, ddx = [torch.empty(N, c * P, device="cuda") for c in (CI, CO, CO, CI)]
s_in, s_out, s_c = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
def ev():
    return torch.cuda.Event(enable_timing=True)
def run(k, verbose):
    bounds = [N * i // k for i in range(k + 1)]
    t0 = ev(); t0.record(s_in); s_out.wait_event(t0)
    marks = []
    xin, dyin = [], []
    for i in range(k):
        a, b = bounds[i], bounds[i + 1]
        e0, e1 = ev(), ev()
        with torch.cuda.stream(s_in):
            e0.record(s_in); dx_[a:b].copy_(hx[a:b], non_blocking=True); e1.record(s_in)
        marks.append(("x%d" % i, e0, e1)); xin.append(e1)
    for i in range(k):
        a, b = bounds[i], bounds[i + 1]
        e0, e1 = ev(), ev()
        with torch.cuda.stream(s_in):
            e0.record(s_in); ddy[a:b].copy_(hdy[a:b], non_blocking=True); e1.record(s_in)
        marks.append(("dy%d" % i, e0, e1)); dyin.append(e1)
    for i in range(k):
        a, b = bounds[i], bounds[i + 1]
        s_out.wait_event(xin[i])
        e0, e1 = ev(), ev()
        with torch.cuda.stream(s_out):
            e0.record(s_out); hy[a:b].copy_(dy_[a:b], non_blocking=True); e1.record(s_out)
        marks.append(("y%d" % i, e0, e1))
    for i in range(k):
        a, b = bounds[i], bounds[i + 1]
        s_out.wait_event(dyin[i])
        e0, e1 = ev(), ev()
        with torch.cuda.stream(s_out):
            e0.record(s_out); hdx[a:b].copy_(ddx[a:b], non_blocking=True); e1.record(s_out)
        marks.append(("dx%d" % i, e0, e1))
    end = ev(); end.record(s_out)
    end.synchronize(); torch.cuda.synchronize()
    tot = t0.elapsed_time(end) * 1e3
    if verbose:
        print(" ".join(f"{n}:{t0.elapsed_time(a) * 1e3:.0f}-{t0.elapsed_time(b) * 1e3:.0f}" for n, a, b in marks))
    return tot
for k in (1, 2, 3, 4, 6, 8):
    for _ in range(3): run(k, False)
    ts = sorted(run(k, False) for _ in range(10))
    print(f"chunks={k}: copies-only {ts[0]:.0f} us (median {ts[5]:.0f})  {4 * N * P * (3 * CI + 2 * CO) / ts[0] / 1e3:.1f} GB/s", flush=True)
    run(k, True)
# reference rates
for name, f in (("H2D 25.2MB alone", lambda: (dx_.copy_(hx, non_blocking=True), ddy.copy_(hdy, non_blocking=True))),
                ("D2H 25.2MB alone", lambda: (hy.copy_(dy_, non_blocking=True), hdx.copy_(ddx, non_blocking=True)))):
    f(); torch.cuda.synchronize()
    a, b = ev(), ev(); a.record(); f(); b.record(); b.synchronize()
    us = a.elapsed_time(b) * 1e3
    print(f"{name}: {us:.0f} us  {25.17e6 / us / 1e3:.1f} GB/s")
