"""Benchmark: DiffMPC fwd+bwd solves/s for the 13-state quadrotor at T=10 (BASELINE.json).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--batch B] [--layout dense|diag]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P bench.py --gpus N --steps K --warmup W

A "step" is one DiffMPC forward (fused iLQR, one kernel) plus one implicit backward
(one kernel) over a batch of B=16384 synthetic hover problems per GPU (BASELINE config 3,
weak scaling: every rank solves its own shard, no data-path collective). Inputs are
larger than L2 (dense C alone is 189 MB), so no explicit L2 flush is needed.

Printed on rank 0 as one JSON line:
  value   whole-job solves/s with inputs resident in HBM (device-timed, max over ranks)
  e2e     the same metric through the public API with pinned HOST buffers: every step
          copies the step's inputs host->device and reads the results device->host
  roofline  the forward kernel (dominant) against the measured FP32 FFMA peak
  cpu_baseline  the C oracle port on this box's host cores (bounded sample)
--impl reference times the reference algorithm on the host cores (the C oracle port;
the reference itself is CPU Python/numba and is not shipped to the GPU box).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DiffMPC fwd+bwd solves/sec (quadrotor, T=10) at 1/2/4/8 B200; per-iter latency"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=16384)
    ap.add_argument("--T", type=int, default=10)
    ap.add_argument("--layout", default="dense", choices=["dense", "diag"])
    ap.add_argument("--dtype", default="f32", choices=["f32", "f64"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(args, rank=0, world=1):
    """Rank `rank`'s contiguous shard (shard.shard_range) of ONE global batch of
    world x batch hover problems (seed 0): the sharding the multi-GPU tests cover."""
    from paper_2605_29155_b200 import DynModel, problems, shard
    model = DynModel.quadrotor(dt=0.05)
    Bg = args.batch * world
    pb = problems.hover_problem(model, Bg, args.T, seed=0)
    lo, hi = shard.shard_range(Bg, rank, world)
    return pb.slice(lo, hi)


def config(args, world):
    return {"workload": "quadrotor13 DiffMPC fwd+bwd (hover problems, K_max=10, conv_tol=1e-6)",
            "n_state": 13, "n_ctrl": 4, "T": args.T, "batch_per_gpu": args.batch,
            "global_batch": args.batch * world, "cost_layout": args.layout,
            "parallelism": f"batch-sharded x{world} (no data-path collective)",
            "l2": "inputs > L2 (dense C 189 MB per step), no flush needed"
            if args.layout == "dense" else "inputs < L2; L2 flushed between steps"}


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # wait for the first sample: nvidia-smi's NVML start-up on a fresh box can stall
            # the GPU for tens of ms, which must not land inside a timed region
            t0 = time.time()
            while not self.samples and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for ln in self.proc.stdout:
            p = [x.strip() for x in ln.split(",")]
            if len(p) >= 9:
                self.samples.append(p)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        mx = [float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[5 + i].strip() == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


# --------------------------------------------------------------------------- CPU legs
def cpu_oracle_rate(pb, seconds=12.0, threads=None, dLdU=None):
    """Oracle port (C, float64, pthreads over problems) fwd+bwd solves/s on a bounded sample."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    threads = threads or len(os.sched_getaffinity(0))
    n = min(pb.B, max(64, 64 * threads))
    C = pb.dense_C()[:n]
    sl = slice(0, n)
    done, t0 = 0, time.perf_counter()
    while True:
        o = oracle.forward(pb.model, pb.settings, pb.x0[sl], C, pb.c[sl], pb.U_warm[sl], threads=threads)
        dU = np.zeros((n, pb.settings.T, pb.model.n_u))
        dU[:, 0, :] = 1.0
        oracle.backward(pb.model, pb.settings, C, pb.c[sl], o["X"], o["U"], None, dU, threads=threads,
                        want_theta=False)
        done += n
        el = time.perf_counter() - t0
        if el >= seconds:
            break
    return done / el, threads, f"{done} hover problems (dense C, T={pb.settings.T}) fwd+bwd in {el:.1f} s"


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return 0
    pb = workload(args)
    rates = []
    for _ in range(max(1, args.warmup // 3)):
        cpu_oracle_rate(pb, seconds=2.0)
    for _ in range(args.steps):
        r, thr, sample = cpu_oracle_rate(pb, seconds=6.0 / max(1, args.steps) * 4)
        rates.append(r)
    v = float(np.median(rates))
    line = {"metric": METRIC, "value": v, "unit": "solves/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * args.batch / v, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config(args, 1), "impl": "reference",
            "cpu_baseline": {"value": v, "unit": "solves/s", "cores": thr, "kind": "port", "sample": sample},
            "e2e": {"value": v, "unit": "solves/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "reference algorithm = C restatement of fusedmpc (oracle/, bit-exact vs the reference "
                    "goldens); the reference package itself is CPU Python/numba"}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- our arm
def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2605_29155_b200 import _lib, roofline, solver

    rank, world, local = dist_env()
    # DIFFMPC_DRYRUN_SHARE_GPU=1: every rank on cuda:0 over gloo (exercises the multi-rank
    # path on a one-GPU box; never used for reported numbers)
    share = os.environ.get("DIFFMPC_DRYRUN_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl", **({} if share else {"device_id": dev}))
    dtype = torch.float32 if args.dtype == "f32" else torch.float64
    pb = workload(args, rank, world)
    model, st = pb.model, pb.settings
    B, T, n, m = args.batch, args.T, model.n_x, model.n_u
    Ch = pb.dense_C() if args.layout == "dense" else pb.diag
    host = {"x0": pb.x0, "C": Ch, "c": pb.c, "U_warm": pb.U_warm}
    dLdU_h = np.zeros((B, T, m))
    dLdU_h[:, 0, :] = 1.0  # the AC-MPC layer's seed: dL/du_0 (policy.py:272)
    host["dLdU"] = dLdU_h
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dtype).pin_memory() for k, v in host.items()}
    dev_in = {k: v.to(dev) for k, v in pinned.items()}
    stream = torch.cuda.current_stream()
    flush = None if args.layout == "dense" else torch.empty(int(256e6), dtype=torch.uint8, device=dev)

    def step(inp):
        out = solver.solve_raw(model, st, inp["x0"], inp["C"], inp["c"], inp["U_warm"], dtype=dtype)
        g = solver.backward_raw(model, st, inp["C"], inp["c"], out.X, out.U, None, inp["dLdU"], dtype=dtype)
        return out, g

    # ---- device-resident timing (value) ----
    # Through a SolvePlan (the library's preallocated launch path: outputs, gradients and the
    # workspace allocated once, each call patches the input pointers and enqueues the kernel):
    # the same two kernels per step, with ~10x less host work per call than solve_raw, so a
    # slow or contended host cannot starve the GPU between the timed launches.
    plan = solver.SolvePlan(model, st, B, layout=args.layout, dtype=dtype, device=dev)

    def pstep():
        o = plan.solve(dev_in["x0"], dev_in["C"], dev_in["c"], dev_in["U_warm"])
        return o, plan.backward(None, dev_in["dLdU"])

    clk = ClockSampler(local).__enter__()  # sample clocks from warm-up through the timed region
    for _ in range(args.warmup):
        out, g = pstep()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True),
           torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    launches0 = _lib.launch_count()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    if True:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        for k in range(args.steps):
            if flush is not None:
                flush.zero_()
            e0, e1, e2 = ev[k]
            e0.record(stream)
            out = plan.solve(dev_in["x0"], dev_in["C"], dev_in["c"], dev_in["U_warm"])
            e1.record(stream)
            g = plan.backward(None, dev_in["dLdU"])
            e2.record(stream)
        t_end.record(stream)
        torch.cuda.synchronize()
    clk.__exit__(None, None, None)
    gpu_launches = _lib.launch_count() - launches0
    elapsed_ms = t_start.elapsed_time(t_end)
    fwd_ms = float(np.mean([a.elapsed_time(b) for a, b, _ in ev]))
    bwd_ms = float(np.mean([b.elapsed_time(c) for _, b, c in ev]))
    step_max = float(max(a.elapsed_time(c) for a, _, c in ev))  # a stall inside the timed region shows here
    if world > 1:
        t = torch.tensor([elapsed_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())
    ms_per_step = elapsed_ms / args.steps
    value = world * B / (ms_per_step * 1e-3)
    iters = out.iters.float()  # (identical inputs every step: the last step's counts)
    it_np = out.iters.cpu().numpy()

    # ---- end-to-end through the public API with pinned host buffers ----
    # Every step copies its inputs host->device, solves + differentiates, and copies the
    # results device->host. Steps are issued round-robin on NS streams so the H2D copy of
    # step k+1, the kernels of step k and the D2H copy of step k-1 overlap (the two PCIe
    # directions run on separate copy engines), as a serving loop would stream batches.
    NS = int(os.environ.get("DIFFMPC_E2E_STREAMS", "3"))
    streams = [torch.cuda.Stream(device=dev) for _ in range(NS)]
    res_host = [{"U": torch.empty((B, T, m), dtype=dtype).pin_memory(),
                 "J": torch.empty((B,), dtype=dtype).pin_memory(),
                 "dC": torch.empty(tuple(Ch.shape), dtype=dtype).pin_memory(),
                 "dc": torch.empty((B, T, n + m), dtype=dtype).pin_memory(),
                 "dx0": torch.empty((B, n), dtype=dtype).pin_memory()} for _ in range(NS)]
    h2d = sum(v.numel() * v.element_size() for v in pinned.values())
    d2h = sum(v.numel() * v.element_size() for v in res_host[0].values())

    def e2e_step(k):
        s = streams[k % NS]
        with torch.cuda.stream(s):
            inp = {kk: v.to(dev, non_blocking=True) for kk, v in pinned.items()}
            out, g = step(inp)
            rh = res_host[k % NS]
            rh["U"].copy_(out.U, non_blocking=True)
            rh["J"].copy_(out.J, non_blocking=True)
            rh["dC"].copy_(g.dC, non_blocking=True)
            rh["dc"].copy_(g.dc, non_blocking=True)
            rh["dx0"].copy_(g.dx0, non_blocking=True)

    for k in range(max(2 * NS, args.warmup // 2)):
        e2e_step(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ke = max(3 * NS, args.steps // 2)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for s_ in streams:  # every stream starts after the start marker
        s_.wait_event(a)
    for k in range(ke):
        e2e_step(k)
    for s_ in streams:  # the end marker waits for every stream
        ev_s = torch.cuda.Event()
        ev_s.record(s_)
        stream.wait_event(ev_s)
    b.record(stream)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / ke
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = world * B / (e2e_ms * 1e-3)
    pcie = pcie_bidir_gbs(dev)  # both copy directions at once: the bound of the e2e leg

    # ---- latency path (BASELINE config 2): forward-only at B=1 and B=256 ----
    lat = {}
    if rank == 0:
        for Bl in (1, 256):
            pl = __import__("paper_2605_29155_b200.problems", fromlist=["x"]).hover_problem(model, Bl, T, seed=7)
            Cl = torch.tensor(pl.dense_C() if args.layout == "dense" else pl.diag, dtype=dtype, device=dev)
            xi, ci, ui = (torch.tensor(z, dtype=dtype, device=dev) for z in (pl.x0, pl.c, pl.U_warm))
            plan = solver.SolvePlan(model, pl.settings, Bl, layout=args.layout, dtype=dtype, device=dev,
                                    backward=False)
            for _ in range(5):
                o = plan.solve(xi, Cl, ci, ui)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            reps = 50
            for _ in range(reps):
                o = plan.solve(xi, Cl, ci, ui)
            e1.record(stream)
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / reps
            mx = int(o.iters.max().item())
            # synchronous call through the preallocated plan: host issue + kernel + sync
            t0 = time.perf_counter()
            for _ in range(20):
                plan.solve(xi, Cl, ci, ui)
                torch.cuda.synchronize()
            wall = (time.perf_counter() - t0) / 20 * 1e3
            lat[f"b{Bl}_fwd_ms"] = round(ms, 4)
            lat[f"b{Bl}_per_iter_us"] = round(1e3 * ms / max(1, mx), 2)
            lat[f"b{Bl}_sync_call_ms"] = round(wall, 4)

    # ---- fixed work: conv_tol = 0, every problem runs K_max iterations ----
    import dataclasses
    st0 = dataclasses.replace(st, conv_tol=0.0)
    fx = []
    for k in range(3 + 10):
        e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
        e0.record(stream)
        o0 = solver.solve_raw(model, st0, dev_in["x0"], dev_in["C"], dev_in["c"], dev_in["U_warm"], dtype=dtype)
        e1.record(stream)
        solver.backward_raw(model, st0, dev_in["C"], dev_in["c"], o0.X, o0.U, None, dev_in["dLdU"], dtype=dtype)
        e2.record(stream)
        if k >= 3:
            fx.append((e0, e1, e2))
    torch.cuda.synchronize()
    fx_f = float(np.median([a.elapsed_time(b) for a, b, _ in fx]))
    fx_b = float(np.median([b.elapsed_time(c) for _, b, c in fx]))
    it0 = o0.iters.cpu().numpy()
    fixed = {"value": world * B / ((fx_f + fx_b) * 1e-3), "unit": "solves/s", "forward_ms": fx_f,
             "backward_ms": fx_b, "mean_iters": float(it0.mean()),
             "fwd_tflops": roofline.fwd_flops(n, m, T, it0, len(st.alphas)) / (fx_f * 1e-3) / 1e12,
             "how": "conv_tol=0, K_max=10, same inputs; per-rank device time, median of 10"}

    # ---- the same step in float64 (the reference's precision), device-timed ----
    f64leg = None
    if dtype == torch.float32 and rank == 0:
        d64 = {k: v.to(torch.float64) for k, v in dev_in.items()}
        ev64 = []
        for k in range(3 + 5):
            e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
            e0.record(stream)
            o64 = solver.solve_raw(model, st, d64["x0"], d64["C"], d64["c"], d64["U_warm"], dtype=torch.float64)
            e1.record(stream)
            solver.backward_raw(model, st, d64["C"], d64["c"], o64.X, o64.U, None, d64["dLdU"],
                                dtype=torch.float64)
            e2.record(stream)
            if k >= 3:
                ev64.append((e0, e1, e2))
        torch.cuda.synchronize()
        f64_f = float(np.median([a.elapsed_time(b) for a, b, _ in ev64]))
        f64_b = float(np.median([b.elapsed_time(c) for _, b, c in ev64]))
        f64leg = {"dtype": "f64", "value": B / ((f64_f + f64_b) * 1e-3), "unit": "solves/s",
                  "forward_ms": f64_f, "backward_ms": f64_b,
                  "how": "same inputs and settings, float64 kernels; rank 0, median of 5 after 3 warm-up"}
        del d64, o64

    # ---- the AC-MPC layer's diagonal cost layout, device and end to end (rank 0) ----
    diag_leg = None
    if args.layout == "dense" and rank == 0:
        diag_leg = diag_layout_leg(pb, dtype, dev, max(10, args.steps // 2), max(3, args.warmup // 2))

    # ---- self-check of the timed outputs against the oracle (untimed, bounded sample) ----
    parity = None
    if rank == 0:
        parity = self_check(pb, out, g, dtype, args.layout)

    # ---- roofline of the dominant kernel (the fused forward) ----
    F = roofline.fwd_flops(n, m, T, it_np, len(st.alphas))
    achieved = F / (fwd_ms * 1e-3) / 1e12
    peak, peak_kind = fp32_peak(dev)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"forward_{args.layout}_{args.dtype}")
        except Exception:
            traffic = None
    bytes_fwd = roofline.fwd_bytes(n, m, T, B, diag=args.layout == "diag", elem=4 if dtype == torch.float32 else 8)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "solves/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
                "config": config(args, world),
                "e2e": {"value": e2e_value, "unit": "solves/s", "h2d_bytes_per_step": int(h2d),
                        "d2h_bytes_per_step": int(d2h), "ms_per_step": e2e_ms,
                        "pipeline": f"{NS} streams round-robin (H2D / kernels / D2H overlap)",
                        "pcie_bound": {"bidir_gbs": pcie, "bound_ms": (h2d + d2h) / (pcie * 1e6),
                                       "frac": (h2d + d2h) / (pcie * 1e6) / e2e_ms,
                                       "how": "64 MB pinned H2D + D2H concurrently on two streams, median of 5"}},
                "gpu_launches": int(gpu_launches),
                "launches_per_step": gpu_launches / args.steps,
                "launches_per_ilqr_iteration": (gpu_launches / args.steps - 1) / float(iters.max().item()),
                "forward_ms": fwd_ms, "backward_ms": bwd_ms, "step_ms_max": step_max,
                "mean_iters": float(iters.mean().item()), "max_iters": int(iters.max().item()),
                "latency": lat,
                "fixed_work": dict(fixed, roofline_frac=fixed["fwd_tflops"] / peak),
                "roofline": {"bound": "fp32", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                             "frac": achieved / peak, "traffic": traffic, "kernel": "ilqr_forward_kernel",
                             "traffic_source": "profiles/traffic.json: dram__bytes_read.sum + "
                                               "dram__bytes_write.sum of this kernel from the committed "
                                               "ncu --set full capture (not measured in this run)",
                             "peak_source": peak_kind,
                             "algorithmic_bytes": bytes_fwd,
                             "hbm_gbs": bytes_fwd / (fwd_ms * 1e-3) / 1e9},
                "clocks": clk.summary(),
                "parity": parity,
                "reference_precision": f64leg,
                "diag_layout": diag_leg}
        if not args.no_cpu_baseline and world == 1:
            r, thr, sample = cpu_oracle_rate(pb, seconds=12.0)
            line["cpu_baseline"] = {"value": r, "unit": "solves/s", "cores": thr, "kind": "port",
                                    "sample": sample}
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def diag_layout_leg(pb, dtype, dev, steps, warmup, NS=3):
    """The same problems in the AC-MPC layer's diagonal cost layout (C_t = diag(d_t),
    MpcSolver.solve_diag, policy.py:214-222): device-resident step (L2 flushed between steps:
    the inputs fit in L2) and end to end from pinned host buffers (3-stream pipeline)."""
    import torch

    from paper_2605_29155_b200 import solver

    model, st = pb.model, pb.settings
    B, T, n, m = pb.B, st.T, model.n_x, model.n_u
    dU = np.zeros((B, T, m))
    dU[:, 0, :] = 1.0
    host = {"x0": pb.x0, "C": pb.diag, "c": pb.c, "U_warm": pb.U_warm, "dLdU": dU}
    pinned = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dtype).pin_memory() for k, v in host.items()}
    dev_in = {k: v.to(dev) for k, v in pinned.items()}
    flush = torch.empty(int(256e6), dtype=torch.uint8, device=dev)

    def step(inp):
        out = solver.solve_raw(model, st, inp["x0"], inp["C"], inp["c"], inp["U_warm"], dtype=dtype)
        g = solver.backward_raw(model, st, inp["C"], inp["c"], out.X, out.U, None, inp["dLdU"], dtype=dtype)
        return out, g

    for _ in range(warmup):
        step(dev_in)
    torch.cuda.synchronize()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        step(dev_in)
        b.record()
        ts.append((a, b))
    torch.cuda.synchronize()
    dev_ms = float(np.mean([a.elapsed_time(b) for a, b in ts]))
    streams = [torch.cuda.Stream(device=dev) for _ in range(NS)]
    res = [{"U": torch.empty((B, T, m), dtype=dtype).pin_memory(), "J": torch.empty((B,), dtype=dtype).pin_memory(),
            "dC": torch.empty((B, T, n + m), dtype=dtype).pin_memory(),
            "dc": torch.empty((B, T, n + m), dtype=dtype).pin_memory(),
            "dx0": torch.empty((B, n), dtype=dtype).pin_memory()} for _ in range(NS)]
    h2d = sum(v.numel() * v.element_size() for v in pinned.values())
    d2h = sum(v.numel() * v.element_size() for v in res[0].values())

    def e2e_step(k):
        s_ = streams[k % NS]
        with torch.cuda.stream(s_):
            out, g = step({kk: v.to(dev, non_blocking=True) for kk, v in pinned.items()})
            r = res[k % NS]
            for name, t in (("U", out.U), ("J", out.J), ("dC", g.dC), ("dc", g.dc), ("dx0", g.dx0)):
                r[name].copy_(t, non_blocking=True)

    for k in range(2 * NS):
        e2e_step(k)
    torch.cuda.synchronize()
    main = torch.cuda.current_stream()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for s_ in streams:
        s_.wait_event(a)
    K = max(3 * NS, steps)
    for k in range(K):
        e2e_step(k)
    for s_ in streams:
        e = torch.cuda.Event()
        e.record(s_)
        main.wait_event(e)
    b.record(main)
    torch.cuda.synchronize()
    e2e_ms = a.elapsed_time(b) / K
    return {"value": B / (dev_ms * 1e-3), "unit": "solves/s", "ms_per_step": dev_ms,
            "e2e": {"value": B / (e2e_ms * 1e-3), "unit": "solves/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "how": f"same problems with C_t = diag(d_t) (B,T,nz) in and diag(dC_t) out; rank 0; L2 flushed "
                   f"between device steps; {NS}-stream pipeline end to end"}


def self_check(pb, out, g, dtype, layout, n=512):
    """The timed step's own outputs for the first n problems of the shard vs the C oracle
    on identical (dtype-rounded) inputs: iteration counts, clamp masks and the worst
    per-instance relative error of X, U, J, dC, dc, dx0 (north_star gate: 1e-4 in f32)."""
    import torch

    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle

    from paper_2605_29155_b200 import _abi
    n = min(n, pb.B)
    rnd = (lambda a: np.asarray(a, np.float32).astype(np.float64)) if dtype == torch.float32 else np.asarray
    cost = pb.dense_C()[:n] if layout == "dense" else pb.diag[:n]
    lay = _abi.COST_DENSE if layout == "dense" else _abi.COST_DIAG
    x0, C, c, Uw = rnd(pb.x0[:n]), rnd(cost), rnd(pb.c[:n]), rnd(pb.U_warm[:n])
    dU = np.zeros((n, pb.settings.T, pb.model.n_u))
    dU[:, 0, :] = 1.0
    th = len(os.sched_getaffinity(0))
    ref = oracle.forward(pb.model, pb.settings, x0, C, c, Uw, layout=lay, threads=th)
    rg = oracle.backward(pb.model, pb.settings, C, c, ref["X"], ref["U"], None, dU, layout=lay, threads=th,
                         want_theta=False)

    def rel(a, b):
        a = np.asarray(a, np.float64).reshape(n, -1)
        b = np.asarray(b, np.float64).reshape(n, -1)
        return float((np.abs(a - b).max(1) / np.maximum(1.0, np.abs(b).max(1))).max())

    get = lambda t: t[:n].detach().cpu().numpy()  # noqa: E731
    err = {"X": rel(get(out.X), ref["X"]), "U": rel(get(out.U), ref["U"]),
           "J": rel(get(out.J)[:, None], ref["J"][:, None]), "dC": rel(get(g.dC), rg["dC"]),
           "dc": rel(get(g.dc), rg["dc"]), "dx0": rel(get(g.dx0), rg["dx0"])}
    it_eq = bool(np.array_equal(get(out.iters), ref["iters"]))
    cl_eq = bool(np.array_equal(get(out.clamped).astype(np.uint8), ref["clamped"]))
    tol = 1e-4 if dtype == torch.float32 else 1e-9
    return {"checked": n, "oracle": "oracle/ (C, f64, pinned bit-exact to the reference goldens)",
            "iters_identical": it_eq, "clamp_masks_identical": cl_eq, "max_rel_err": err, "tol": tol,
            "pass": it_eq and cl_eq and max(err.values()) <= tol}


def pcie_bidir_gbs(dev, mb=64, reps=5):
    """Host<->device copy bandwidth with both directions busy (tools/pcie_probe.py)."""
    import torch

    n = mb << 20
    h_in, h_out = torch.empty(n, dtype=torch.uint8).pin_memory(), torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in, d_out = torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2, main = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev), torch.cuda.current_stream(dev)
    ts = []
    for i in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(dev)
        a.record(main)
        for s, (dst, src) in ((s1, (d_in, h_in)), (s2, (h_out, d_out))):
            s.wait_event(a)
            with torch.cuda.stream(s):
                dst.copy_(src, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(s)
            main.wait_event(ev)
        b.record(main)
        torch.cuda.synchronize(dev)
        if i:
            ts.append(a.elapsed_time(b))
    return 2 * n / float(np.median(ts)) / 1e6


def fp32_peak(dev):
    """Measured FP32 FFMA throughput (TFLOP/s) via libdiffmpc's probe kernel."""
    import ctypes

    import torch

    from paper_2605_29155_b200 import _lib
    L = _lib.lib()
    L.diffmpc_probe_ffma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    blocks, iters = sms * 8, 4096
    out = torch.empty(blocks, device=dev)
    s = torch.cuda.current_stream()
    best = 0.0
    for _ in range(4):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        L.diffmpc_probe_ffma(blocks, iters, out.data_ptr(), s.cuda_stream)
        b.record(s)
        torch.cuda.synchronize()
        flops = 2.0 * blocks * 256 * iters * 16 * 8
        best = max(best, flops / (a.elapsed_time(b) * 1e-3) / 1e12)
    return best, "measured FFMA probe (csrc/probe.cu), burst"


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
