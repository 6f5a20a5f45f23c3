"""Diagnose iteration-count flips of the f32 throughput kernel vs the oracle on bench
workloads (development aid): per flipped instance, both J / alpha histories, the per-
iteration relative decrease and each side's convergence decision.

python tools/flip_diag.py [hover|random] [dense|diag]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests"), os.path.join(ROOT, "oracle")]
import numpy as np  # noqa: E402
import torch  # noqa: E402

import parity_util as pu  # noqa: E402
import test_gpu_bench_parity as tb  # noqa: E402
from paper_2605_29155_b200 import solver  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "random"
layout = sys.argv[2] if len(sys.argv) > 2 else "dense"
pb = tb.workload(name)
(x0, C, c, Uw, dX, dU), ref, refg = tb.oracle_run(name, layout, "f32", "layer")
out = solver.solve_raw(pb.model, pb.settings, x0, C, c, Uw, dtype=torch.float32, kernel="throughput")
torch.cuda.synchronize()
it = pu.as_np(out.iters)
flips = np.nonzero(it != ref["iters"])[0]
print("flips", flips.tolist())
Jh, ah = pu.as_np(out.J_hist).astype(np.float64), pu.as_np(out.alpha_hist)
ct = pb.settings.conv_tol
for i in flips[:10]:
    print(f"--- instance {i}: gpu iters {it[i]} oracle iters {ref['iters'][i]}")
    for k in range(pb.settings.K_max + 1):
        jg, jo = Jh[i, k], ref["J_hist"][i, k]
        rg = abs(Jh[i, k - 1] - jg) / max(1, abs(Jh[i, k - 1])) if k else float("nan")
        ro = abs(ref["J_hist"][i, k - 1] - jo) / max(1, abs(ref["J_hist"][i, k - 1])) if k else float("nan")
        a = f"alpha gpu {ah[i, k - 1]:.3g} ora {ref['alpha_hist'][i, k - 1]:.3g}" if k else ""
        print(f"  k={k:2d} J gpu {jg:.9e} ora {jo:.9e}  rel/conv_tol gpu {rg / ct:10.4f} ora {ro / ct:10.4f} {a}")
    e = pu.rel_err(pu.as_np(out.U)[i:i + 1], ref["U"][i:i + 1])[0]
    print(f"  final U rel err {e:.2e}; clamped gpu {int(pu.as_np(out.clamped)[i].sum())} ora {int(ref['clamped'][i].sum())}")

# the instance with the largest J-history error among those with identical counts
same = (it == ref["iters"]) & (ref["fail_t"] < 0)
e = pu.rel_err(Jh, ref["J_hist"])
e[~same] = 0
for i in np.argsort(-e)[:3]:
    print(f"--- J_hist err {e[i]:.2e} instance {i}: iters {it[i]}")
    print("  gpu", " ".join(f"{v:.7e}" for v in Jh[i, :it[i] + 1]))
    print("  ora", " ".join(f"{v:.7e}" for v in ref["J_hist"][i, :it[i] + 1]))
    print("  alpha gpu", ah[i, :it[i]].tolist(), "ora", ref["alpha_hist"][i, :it[i]].tolist())
