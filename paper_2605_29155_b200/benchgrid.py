"""Latency grid in the reference's bench CSV format.

Mirrors batchexec.latency_probe / write_latency_csv
(/root/reference/pkg/src/fusedmpc/batchexec.py:39, 242-293): hover problems with
K_max = K and conv_tol = 0 (fixed work), one warm-up round per cell, median wall times
of the array-level forward and backward calls. The columns are exactly the report tool's
BENCH schema (reports/src/mpcreports/schemas.py:9), so ``mpc-report latency_bars`` can
render the B200 rows (mode "b200") beside the reference's "fused" / "naive" CPU rows.

Timing semantics match the reference's array API: inputs are host numpy arrays and the
call returns host results (solution / gradients copied back), so each wall time includes
the host<->device copies; ``dispatches`` counts the library's kernel launches (one
forward, one backward).

    python -m paper_2605_29155_b200.benchgrid --B 1 64 1024 16384 --T 10 --out bench.csv
"""

from __future__ import annotations

import argparse
import csv
import statistics
import time

import numpy as np

from .dynamics import DynModel
from .errors import ConfigError

LATENCY_CSV_HEADER = ["mode", "B", "T", "K", "forward_ms", "backward_ms", "dispatches"]
MODE = "b200"


def latency_probe(B_list, T_list, reps=10, K=10, seed=0, model=None, layout="dense"):
    import torch

    from . import _lib, problems, solver

    if reps < 1:
        raise ConfigError(f"reps must be >= 1, got {reps}")
    model = model or DynModel.planar_quadrotor(dt=0.05)
    rows = []
    for B in B_list:
        for T in T_list:
            pb = problems.hover_problem(model, B, T, seed=seed, K_max=K, conv_tol=0.0)
            C = pb.dense_C() if layout == "dense" else pb.diag
            dU = np.zeros((B, T, model.n_u))
            dU[:, 0, :] = 1.0  # the unit seed dL/du_0 of batchexec._unit_seeds

            def fwd():
                out = solver.solve_raw(model, pb.settings, pb.x0, C, pb.c, pb.U_warm, dtype=torch.float64)
                host = (solver.to_numpy(out.X), solver.to_numpy(out.U), solver.to_numpy(out.J))
                return out, host

            def bwd(out):
                g = solver.backward_raw(model, pb.settings, out.C, out.c, out.X, out.U, None, dU, dtype=torch.float64)
                return solver.to_numpy(g.dC), solver.to_numpy(g.dc), solver.to_numpy(g.dx0)

            out, _ = fwd()  # warm-up round (excluded)
            bwd(out)
            torch.cuda.synchronize()
            ft, bt = [], []
            l0 = _lib.launch_count()
            for _ in range(reps):
                t0 = time.perf_counter()
                out, _ = fwd()
                ft.append(time.perf_counter() - t0)
                t0 = time.perf_counter()
                bwd(out)
                bt.append(time.perf_counter() - t0)
            rows.append({"mode": MODE, "B": B, "T": T, "K": K, "forward_ms": 1e3 * statistics.median(ft),
                         "backward_ms": 1e3 * statistics.median(bt),
                         "dispatches": (_lib.launch_count() - l0) // reps})
    return rows


def write_latency_csv(rows, path):
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=LATENCY_CSV_HEADER)
        w.writeheader()
        for r in rows:
            w.writerow(r)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--B", type=int, nargs="+", default=[1, 64, 1024, 16384])
    ap.add_argument("--T", type=int, nargs="+", default=[10])
    ap.add_argument("--K", type=int, default=10)
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--model", default="planar", choices=["planar", "quad13"])
    ap.add_argument("--out", default="bench.csv")
    a = ap.parse_args()
    model = DynModel.planar_quadrotor(dt=0.05) if a.model == "planar" else DynModel.quadrotor(dt=0.05)
    rows = latency_probe(a.B, a.T, a.reps, a.K, model=model)
    write_latency_csv(rows, a.out)
    for r in rows:
        print(r)


if __name__ == "__main__":
    main()
