"""Measured parity table (markdown): every golden case x layout x dtype x forward mapping,
plus bench.py's own B=16384 workloads, GPU kernels vs the reference goldens / the C
oracle on identical inputs. Worst per-instance relative errors per tensor, iteration-count
flips (with the oracle-side decision margin), mask / flag mismatches.

python tools/parity_report.py [out.md]      (runs on the GPU box; tests/parity_util.py)
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import golden_util as gu  # noqa: E402
import parity_util as pu  # noqa: E402
from paper_2605_29155_b200 import solver  # noqa: E402

rows = []


def fmt(rep, brep):
    e = dict(rep["err"])
    e.update({k: v for k, v in brep["err"].items()})
    keys = ("X", "U", "J", "K", "k", "J_hist", "dC", "dc", "dx0", "dX", "dU")
    errs = " | ".join(f"{e[k]:.1e}" if k in e else "-" for k in keys)
    flips = len(rep["flips"])
    fl = f"{flips}" + (f" (margins {', '.join(f'{m:+.1e}' for m in rep['flip_margins'][:4])})" if flips else "")
    mism = (rep["clamp_mismatch"] + rep["converged_mismatch"] + rep["alpha_hist_mismatch"] + rep["fail_mismatch"]
            + rep["diverged_mismatch"] + brep["bfail_mismatch"])
    return f"{fl} | {mism} | {errs}"


def golden_rows():
    for name in gu.SOLVE_CASES:
        g = gu.load(name)
        for layout in g.layouts():
            for dtype in (torch.float64, torch.float32):
                for kernel in ("throughput", "latency"):
                    out = solver.solve_raw(g.model, g.settings, g["x0"], g.cost(layout), g["c"], g["U_warm"],
                                           dtype=dtype, kernel=kernel)
                    rep = pu.compare_forward(out, g.d, dtype, g.settings.conv_tol)
                    res = solver.backward_raw(g.model, g.settings, g.cost(layout), g["c"], g["X"], g["U"],
                                              g["dLdX"], g["dLdU"], dtype=dtype, want_traj=True)
                    ok = (g["fail_t"] < 0) & (g["diverged"] == 0)
                    brep = pu.compare_backward(res, g.d, dtype, ok, layout_diag=bool(layout))
                    fail_ok = ok | (g["bfail_t"] >= 0)
                    brep["bfail_mismatch"] = int((pu.as_np(res.fail_t)[fail_ok] != g["bfail_t"][fail_ok]).sum())
                    tag = "conv_tol=0 (counts not gated)" if g.settings.conv_tol == 0 else ""
                    rows.append(f"| {name} {tag} | {'diag' if layout else 'dense'} | {str(dtype)[6:]} | {kernel} | "
                                f"{g.B} | {fmt(rep, brep)} |")
                    print(rows[-1], flush=True)


def bench_rows():
    import test_gpu_bench_parity as tb

    for name, layout in tb.CASES:
        for dt_name in ("f32", "f64"):
            dtype = torch.float32 if dt_name == "f32" else torch.float64
            pb = tb.workload(name)
            (x0, C, c, Uw, dX, dU), ref, refg = tb.oracle_run(name, layout, dt_name, "layer")
            out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=dtype, kernel="throughput")
            g = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, dX, dU, dtype=dtype,
                                    want_traj=True)
            rep = pu.compare_forward(out, ref, dtype, pb.settings.conv_tol)
            same = (pu.as_np(out.iters) == ref["iters"]) & (ref["fail_t"] < 0)
            brep = pu.compare_backward(g, refg, dtype, same, layout_diag=(layout == "diag"))
            rows.append(f"| bench {name} (oracle) | {layout} | {str(dtype)[6:]} | "
                        f"throughput | {pb.B} | {fmt(rep, brep)} |")
            print(rows[-1], flush=True)


if __name__ == "__main__":
    out_path = sys.argv[1] if len(sys.argv) > 1 else None
    bench_rows()
    golden_rows()
    hdr = ("| case | layout | dtype | forward kernel | B | count flips | mask/flag mismatches | "
           "X | U | J | K | k | J_hist | dC | dc | dx0 | dX | dU |\n|" + "---|" * 18)
    txt = ("# Parity, measured on B200 (tools/parity_report.py)\n\nWorst per-instance relative error "
           "max|a-b| / max(1, max|b|) per tensor; gate 1e-4 (f32) / 1e-9 (f64). Goldens: the unmodified "
           "reference (tests/golden/); bench rows: the C oracle on identical (dtype-rounded) inputs, "
           "B=16384, backward seeded with dL/du_0 = 1 as bench.py times it. Mask/flag mismatches = clamp "
           "masks + converged + accepted step sizes + failure + divergence + backward failure stage.\n\n"
           + hdr + "\n" + "\n".join(rows) + "\n")
    if out_path:
        open(out_path, "w").write(txt)
    else:
        print(txt)
