"""BASELINE config 5: horizon / batch sweep of the DiffMPC fwd+bwd step on one B200, with the
CPU oracle port timed on the host cores at each horizon.

    python tools/sweep.py [--T 5 10 20 40] [--B 256 1024 4096 16384 65536 131072] [--layout dense]

Problems are the 13-state hover batch (problems.hover_problem semantics: x0 drawn with the
same seeded generator, diagonal weights, hover reference), built directly on the device so
the largest cases (131072 x T=40 dense C = 6 GB) need no host staging. Device time per step
(CUDA events, median of reps after warm-up) -> solves/s and the forward's roofline fraction
against the measured FFMA peak. One JSON line per case, then a markdown table.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [os.environ.get("DIFFMPC_PKG_ROOT", ROOT), os.path.join(ROOT, "oracle")]  # env: A/B another copy

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2605_29155_b200 import DynModel, problems, roofline, solver  # noqa: E402


def device_problem(model, B, T, layout, dev, seed=0):
    small = problems.hover_problem(model, B, 1, seed=seed)  # x0 + weights (host, tiny)
    st = problems.hover_problem(model, 1, T, seed=seed).settings
    d = torch.tensor(small.diag[0, 0], dtype=torch.float32, device=dev)
    c1 = torch.tensor(small.c[0, 0], dtype=torch.float32, device=dev)
    nz = d.numel()
    diag = d.expand(B, T, nz).contiguous()
    C = torch.diag_embed(diag) if layout == "dense" else diag
    c = c1.expand(B, T, nz).contiguous()
    x0 = torch.tensor(small.x0, dtype=torch.float32, device=dev)
    Uw = torch.tensor(small.U_warm[0, 0], dtype=torch.float32, device=dev).expand(B, T, model.n_u).contiguous()
    return st, x0, C, c, Uw


def time_case(model, B, T, layout, dev, budget_s=1.5):
    st, x0, C, c, Uw = device_problem(model, B, T, layout, dev)
    dLdU = torch.zeros((B, T, model.n_u), device=dev)
    dLdU[:, 0] = 1.0
    out = solver.solve_raw(model, st, x0, C, c, Uw)
    g = solver.backward_raw(model, st, C, c, out.X, out.U, None, dLdU)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        out = solver.solve_raw(model, st, x0, C, c, Uw)
        g = solver.backward_raw(model, st, C, c, out.X, out.U, None, dLdU)
    torch.cuda.synchronize()
    per = (time.perf_counter() - t0) / 2
    reps = int(min(50, max(3, budget_s / max(per, 1e-4))))
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(reps)]
    for e0, e1, e2 in ev:
        e0.record()
        out = solver.solve_raw(model, st, x0, C, c, Uw)
        e1.record()
        g = solver.backward_raw(model, st, C, c, out.X, out.U, None, dLdU)
        e2.record()
    torch.cuda.synchronize()
    fwd = float(np.median([a.elapsed_time(b) for a, b, _ in ev]))
    bwd = float(np.median([b.elapsed_time(c_) for _, b, c_ in ev]))
    it = out.iters.cpu().numpy()
    del g
    F = roofline.fwd_flops(model.n_x, model.n_u, T, it, len(st.alphas))
    return {"T": T, "B": B, "layout": layout, "fwd_ms": fwd, "bwd_ms": bwd, "solves_per_s": B / ((fwd + bwd) * 1e-3),
            "mean_iters": float(it.mean()), "max_iters": int(it.max()),
            "fwd_tflops": F / (fwd * 1e-3) / 1e12, "reps": reps}


def cpu_rate(model, T, seconds=3.0):
    import oracle
    threads = len(os.sched_getaffinity(0))
    n = 64 * threads
    pb = problems.hover_problem(model, n, T, seed=0)
    C = pb.dense_C()
    done, t0 = 0, time.perf_counter()
    while True:
        o = oracle.forward(model, pb.settings, pb.x0, C, pb.c, pb.U_warm, threads=threads)
        dU = np.zeros((n, T, model.n_u))
        dU[:, 0] = 1.0
        oracle.backward(model, pb.settings, C, pb.c, o["X"], o["U"], None, dU, threads=threads, want_theta=False)
        done += n
        if time.perf_counter() - t0 >= seconds:
            break
    return done / (time.perf_counter() - t0), threads


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--T", type=int, nargs="+", default=[5, 10, 20, 40])
    ap.add_argument("--B", type=int, nargs="+", default=[256, 1024, 4096, 16384, 65536, 131072])
    ap.add_argument("--layout", default="dense", choices=["dense", "diag"])
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda")
    model = DynModel.quadrotor(dt=0.05)
    sys.path.insert(0, ROOT)
    from bench import fp32_peak
    peak, _ = fp32_peak(dev)
    # CPU samples first (a 3 s host phase would let the GPU clocks drop between cases),
    # then warm the GPU (clocks, module load, allocator) before the first timed case
    cpus = {T: (None if args.no_cpu else cpu_rate(model, T)) for T in args.T}
    for _ in range(3):
        time_case(model, 16384, 10, args.layout, dev, budget_s=0.3)
    rows = []
    for T in args.T:
        cpu = cpus[T]
        for B in args.B:
            r = time_case(model, B, T, args.layout, dev)
            r["roofline_frac"] = r["fwd_tflops"] / peak
            if cpu:
                r["cpu_solves_per_s"], r["cpu_threads"] = cpu
            rows.append(r)
            print(json.dumps(r), flush=True)
            torch.cuda.empty_cache()
    print(f"\nFFMA peak {peak:.1f} TFLOP/s (measured)\n")
    print("| T | B | fwd ms | bwd ms | solves/s | mean it | fwd TFLOP/s | frac | CPU solves/s (threads) |")
    print("|---|---|---|---|---|---|---|---|---|")
    for r in rows:
        cpu = f"{r['cpu_solves_per_s']:.0f} ({r['cpu_threads']})" if "cpu_solves_per_s" in r else "-"
        print(f"| {r['T']} | {r['B']} | {r['fwd_ms']:.3f} | {r['bwd_ms']:.3f} | {r['solves_per_s']:.3g} | "
              f"{r['mean_iters']:.2f} | {r['fwd_tflops']:.2f} | {100 * r['roofline_frac']:.1f}% | {cpu} |")


if __name__ == "__main__":
    main()
