"""The N>1 paths with the REAL CUDA kernels, on the one-GPU box: two ranks share cuda:0 over
gloo (DIFFMPC_DRYRUN_SHARE_GPU's arrangement; NCCL refuses two ranks on one device).

  * sharded solve: each rank solves its shard_range slice of one global batch (forward +
    backward kernels) and the all-gathered result equals the single-process solve bit for
    bit (the throughput mapping is batch-size invariant) — SURVEY.md §8(e);
  * bench.py under torchrun --nproc-per-node 2: the JSON line of the sharded benchmark;
  * data-parallel PPO with the graphed minibatch step and the flat-bucket all-reduce:
    replicas identical and equal to one process stepping on the whole minibatch.
"""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _solve(pb, C, lo=None, hi=None):
    from paper_2605_29155_b200 import solver

    sl = slice(lo, hi)
    out = solver.solve_raw(pb.model, pb.settings, pb.x0[sl], C[sl], pb.c[sl], pb.U_warm[sl], dtype=torch.float32,
                           device="cuda:0", kernel="throughput")
    dU = torch.zeros_like(out.U)
    dU[:, 0] = 1.0
    g = solver.backward_raw(pb.model, pb.settings, out.C, out.c, out.X, out.U, None, dU, dtype=torch.float32)
    return {"U": out.U, "X": out.X, "J": out.J, "iters": out.iters.to(torch.int64), "dC": g.dC, "dx0": g.dx0}


def _problem(B):
    from paper_2605_29155_b200 import DynModel, problems
    pb = problems.random_problem(DynModel.quadrotor(), B, 10, seed=77)
    return pb, pb.dense_C()


def _shard_worker(rank, world, port, B, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_29155_b200 import shard

    pb, C = _problem(B)
    lo, hi = shard.shard_range(B, rank, world)
    res = _solve(pb, C, lo, hi)
    torch.cuda.synchronize()
    full = {k: shard.all_gather_batch(v.cpu(), B) for k, v in res.items()}
    if rank == 0:
        q.put({k: v.numpy() for k, v in full.items()})
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_sharded_solve_with_cuda_kernels():
    B, world = 999, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_shard_worker, args=(r, world, port, B, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    pb, C = _problem(B)
    ref = _solve(pb, C)
    for k, v in ref.items():
        np.testing.assert_array_equal(got[k], v.cpu().numpy(), err_msg=k)


def test_bench_runs_sharded_under_torchrun():
    env = dict(os.environ, DIFFMPC_DRYRUN_SHARE_GPU="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--batch", "2048", "--no-cpu-baseline"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 prints the one line
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["config"]["global_batch"] == 4096
    assert line["parity"]["pass"] and line["gpu_launches"] == 2 * 3
    assert line["value"] > 0 and line["e2e"]["value"] > 0


def _ppo_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2605_29155_b200 import ppo
    sd, batches, cfg, model, st = _ppo_setup()
    b, opt, solver = _ppo_bundle(sd, model, st)
    red = ppo.GradAllReduce(b.parameters())
    lo, hi = rank * 64, (rank + 1) * 64  # this rank's half of every 128-sample minibatch
    gstep = ppo.GraphedMinibatchStep(b, opt, {k: v[lo:hi] for k, v in batches[0].items()}, cfg, solver, reducer=red)
    assert not gstep.in_graph  # gloo: the all-reduce runs between the replay and the clipping
    for bt in batches:
        gstep({k: v[lo:hi] for k, v in bt.items()})
    flat = torch.cat([p.detach().reshape(-1) for p in b.parameters()]).cpu()
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat)
    if rank == 0:
        q.put((parts[0].numpy(), parts[1].numpy()))
    dist.barrier()
    dist.destroy_process_group()


def _ppo_setup():
    from paper_2605_29155_b200 import DynModel, SolveSettings, ppo
    from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle

    model = DynModel.quadrotor(dt=0.05)
    st = SolveSettings(T=5, u_min=0.0, u_max=float(model.params[0] * model.params[-1]))
    torch.manual_seed(0)
    b = PolicyBundle("ac_mpc", 13, model, st, CostHeadScaling.for_model(model, 13), hidden=(64, 64))
    sd = {k: v.clone() for k, v in b.state_dict().items()}
    g = torch.Generator().manual_seed(4)
    batches = []
    for _ in range(3):
        x = 0.3 * torch.randn(128, 13, generator=g)
        x[:, 3] += 1.0
        batches.append({"obs": x.clone(), "actions": 1.5 + torch.randn(128, 4, generator=g),
                        "old_log_probs": torch.randn(128, generator=g) - 3.0,
                        "advantages": torch.randn(128, generator=g), "returns": torch.randn(128, generator=g),
                        "x_init": x.clone(), "U_warm": torch.full((128, 5, 4), 1.47)})
    batches = [{k: v.cuda() for k, v in bt.items()} for bt in batches]
    return sd, batches, ppo.TrainConfig(), model, st


def _ppo_bundle(sd, model, st):
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle

    b = PolicyBundle("ac_mpc", 13, model, st, CostHeadScaling.for_model(model, 13), hidden=(64, 64))
    b.load_state_dict(sd)
    b = b.cuda()
    return b, torch.optim.Adam(b.parameters(), lr=3e-4), MpcSolver(model, st, device="cuda:0")


def test_two_rank_graphed_ppo_step_with_cuda_kernels():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_ppo_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    p0, p1 = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    np.testing.assert_array_equal(p0, p1)  # replicas identical after every step
    from paper_2605_29155_b200 import ppo
    sd, batches, cfg, model, st = _ppo_setup()
    b, opt, solver = _ppo_bundle(sd, model, st)
    for bt in batches:  # one process, whole minibatches: mean of the two half means
        ppo.minibatch_step(b, opt, bt, cfg, solver)
    ref = torch.cat([p.detach().reshape(-1) for p in b.parameters()]).cpu().numpy()
    np.testing.assert_allclose(p0, ref, rtol=1e-4, atol=1e-5)
