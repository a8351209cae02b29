"""Full-batch fp64 reference of the SCC operator in torch, for parity checks
at BASELINE sizes where the scalar oracle would take minutes.

Same semantics as the reference (kernel.cpp:29-181): filters are grouped by
window start, start(oc) = (oc*shift) mod c_in (cycle.cpp:9-26), and each group
is one fp64 GEMM over exactly its gw-channel window (no dense padding, so the
largest C5 shape costs the band's own FLOPs).  Only the summation ORDER
differs from the oracle (fp64 GEMM vs the reference's sequential loops), i.e.
~1e-15 relative -- far below the 1e-5 / 1e-4 fp32 bars.  Pinned against the
oracle by tests/test_oracle.py::test_fp64_class_gemm_reference_matches_oracle.
Test infrastructure only.
"""
import torch


def starts(c_in, c_out, shift):
    return [(oc * shift) % c_in for oc in range(c_out)]


def scc_fp64(c_in, c_out, gw, shift, x, w, b, dy):
    """x [N, c_in, H, W], w [c_out*gw], b [c_out] or None, dy [N, c_out, H, W]
    (any float dtype / device) -> fp64 (y, dx, dw, db)."""
    dev = x.device
    n, _, h, wd = x.shape
    p = h * wd
    x64 = x.double().reshape(n, c_in, p)
    dy64 = dy.double().reshape(n, c_out, p)
    w64 = w.double().reshape(c_out, gw)
    st = starts(c_in, c_out, shift)
    groups = {}
    for oc, s in enumerate(st):
        groups.setdefault(s, []).append(oc)
    y = torch.empty(n, c_out, p, dtype=torch.float64, device=dev)
    dx = torch.zeros(n, c_in, p, dtype=torch.float64, device=dev)
    dw = torch.empty(c_out, gw, dtype=torch.float64, device=dev)
    for s, ocs in groups.items():
        oi = torch.tensor(ocs, device=dev)
        ii = (s + torch.arange(gw, device=dev)) % c_in
        ws = w64.index_select(0, oi)                      # [m, gw]
        xs = x64.index_select(1, ii)                      # [N, gw, P]
        dys = dy64.index_select(1, oi)                    # [N, m, P]
        y[:, oi] = torch.matmul(ws, xs)
        dx.index_add_(1, ii, torch.matmul(ws.t(), dys))
        dw[oi] = torch.einsum("nmp,nkp->mk", dys, xs)
        del xs, dys
    if b is not None:
        y += b.double().view(1, c_out, 1)
    db = dy64.sum(dim=(0, 2)) if b is not None else None
    return (y.view(n, c_out, h, wd), dx.view(n, c_in, h, wd), dw.reshape(-1), db)
