"""Per-case parity table: GPU kernels vs the reference goldens (development aid)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import numpy as np, torch
import golden_util as gu
from paper_2605_29155_b200 import solver

def rel(a, b):
    a = np.asarray(a, float).reshape(a.shape[0], -1); b = np.asarray(b, float).reshape(b.shape[0], -1)
    return np.abs(a - b).max(1) / np.maximum(1.0, np.abs(b).max(1))

for name in gu.SOLVE_CASES:
    g = gu.load(name)
    for layout in g.layouts():
        for dtype in (torch.float64, torch.float32):
            out = solver.solve_raw(g.model, g.settings, g["x0"], g.cost(layout), g["c"], g["U_warm"], dtype=dtype)
            it = out.iters.cpu().numpy(); flips = np.nonzero(it != g["iters"])[0]
            ok = (g["fail_t"] < 0) & (g["diverged"] == 0) & (it == g["iters"])
            eX = rel(out.X.cpu().numpy()[ok], g["X"][ok]).max(initial=0)
            eU = rel(out.U.cpu().numpy()[ok], g["U"][ok]).max(initial=0)
            J = out.J.cpu().numpy(); eJ = (np.abs(J - g["J"]) / np.maximum(1, np.abs(g["J"])))[ok].max(initial=0)
            cm = (out.clamped.cpu().numpy().astype(np.uint8)[ok] != g["clamped"][ok]).any(axis=(1, 2)).sum()
            cv = (out.converged.cpu().numpy().astype(np.uint8) != g["converged"])[ok].sum()
            ft = (out.fail_t.cpu().numpy() != g["fail_t"]).sum()
            dv = (out.diverged.cpu().numpy().astype(np.uint8) != g["diverged"]).sum()
            res = solver.backward_raw(g.model, g.settings, g.cost(layout), g["c"], g["X"], g["U"], g["dLdX"], g["dLdU"], dtype=dtype)
            bok = g["bfail_t"] < 0
            eg = max(rel(res.dC.cpu().numpy()[bok], g.dC_in(layout)[bok]).max(initial=0),
                     rel(res.dc.cpu().numpy()[bok], g["dc"][bok]).max(initial=0),
                     rel(res.dx0.cpu().numpy()[bok], g["dx0"][bok]).max(initial=0))
            bf = (res.fail_t.cpu().numpy() != g["bfail_t"]).sum()
            extra = ""
            if len(flips):
                extra = " flips:" + ",".join(f"{i}({g['iters'][i]}->{it[i]})" for i in flips[:6])
            print(f"{name:20s} {'diag ' if layout else 'dense'} {str(dtype)[6:]:8s} B={g.B:3d} flips={len(flips):2d} "
                  f"X {eX:.1e} U {eU:.1e} J {eJ:.1e} clampΔ {cm} convΔ {cv} failΔ {ft} divΔ {dv} | grad {eg:.1e} bfailΔ {bf}{extra}", flush=True)
