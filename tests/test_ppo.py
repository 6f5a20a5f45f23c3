"""PPO plumbing around the DiffMPC layer.

CPU: gae against a loop restatement of trainer.py:66-91, and the world_size-2 gloo path
of the data-parallel update (one flat gradient all-reduce per minibatch) against a
single-process update on the full minibatch, in the solver-free ac_mlp mode.
GPU: the ac_mpc minibatch step through the B200 layer (ratio 1 at the trust-region
centre, gradients reach the cost actor)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2605_29155_b200 import DynModel, SolveSettings
from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle
from paper_2605_29155_b200 import ppo


def _gae_ref(rewards, values, dones, gamma, lam, last_values):
    S = rewards.shape[0]
    adv = np.zeros_like(rewards)
    next_adv = np.zeros_like(last_values)
    next_val = last_values
    for s in range(S - 1, -1, -1):
        nt = 1.0 - dones[s]
        delta = rewards[s] + gamma * next_val * nt - values[s]
        next_adv = delta + gamma * lam * nt * next_adv
        adv[s] = next_adv
        next_val = values[s]
    return adv, adv + values


def test_gae_matches_loop_restatement():
    rng = np.random.default_rng(0)
    r, v = rng.normal(size=(7, 5)), rng.normal(size=(7, 5))
    d = (rng.random((7, 5)) < 0.2).astype(float)
    lv = rng.normal(size=5)
    a, ret = ppo.gae(r, v, d, 0.99, 0.95, lv)
    a2, ret2 = _gae_ref(r, v, d, 0.99, 0.95, lv)
    np.testing.assert_array_equal(a.numpy(), a2)
    np.testing.assert_array_equal(ret.numpy(), ret2)


def _bundle(mode="ac_mlp", seed=0):
    torch.manual_seed(seed)
    model = DynModel.quadrotor(dt=0.05)
    st = SolveSettings(T=4, u_min=0.0, u_max=model.params[0] * model.params[-1])
    return PolicyBundle(mode, 13, model, st, CostHeadScaling.for_model(model, 13), hidden=(32, 32)), model, st


def _buffer(n, model, T, seed=1):
    g = torch.Generator().manual_seed(seed)
    return {"obs": torch.randn(n, 13, generator=g), "actions": torch.rand(n, 4, generator=g) * 5,
            "log_probs": torch.randn(n, generator=g) - 3, "advantages": torch.randn(n, generator=g),
            "returns": torch.randn(n, generator=g)}


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, model, st = _bundle()
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=64, sgd_epochs=2, normalize_advantages=False)
    opt = torch.optim.Adam(b.parameters(), lr=1e-3)
    red = ppo.GradAllReduce(b.parameters())
    ppo.ppo_update(_buffer(128, model, st.T), b, opt, cfg, generator=torch.Generator().manual_seed(3),
                   reducer=red, rank=rank, world=world)
    flat = torch.cat([p.detach().reshape(-1) for p in b.parameters()])
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat)
    if rank == 0:
        q.put((parts[0].numpy(), parts[1].numpy(), red.nbytes))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_update_matches_single_process():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    p0, p1, nbytes = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    np.testing.assert_array_equal(p0, p1)  # replicas stay identical
    # single process, full minibatches: the mean of the two shard means is the full mean
    b, model, st = _bundle()
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=64, sgd_epochs=2, normalize_advantages=False)
    opt = torch.optim.Adam(b.parameters(), lr=1e-3)
    ppo.ppo_update(_buffer(128, model, st.T), b, opt, cfg, generator=torch.Generator().manual_seed(3))
    ref = torch.cat([p.detach().reshape(-1) for p in b.parameters()]).numpy()
    np.testing.assert_allclose(p0, ref, rtol=1e-5, atol=1e-6)
    assert nbytes == 4 * sum(p.numel() for p in b.parameters())


def _worker_sharded(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    b, model, st = _bundle()
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=64, sgd_epochs=2)
    opt = torch.optim.Adam(b.parameters(), lr=1e-3)
    red = ppo.GradAllReduce(b.parameters())
    # every rank trains on its OWN buffer (its environments' transitions)
    m = ppo.ppo_update(_buffer(96, model, st.T, seed=10 + rank), b, opt, cfg,
                       generator=torch.Generator().manual_seed(3), reducer=red, rank=rank, world=world,
                       data="sharded")
    flat = torch.cat([p.detach().reshape(-1) for p in b.parameters()])
    parts = [torch.empty_like(flat) for _ in range(world)]
    dist.all_gather(parts, flat)
    if rank == 0:
        q.put((parts[0].numpy(), parts[1].numpy(), m["samples_trained"]))
    dist.barrier()
    dist.destroy_process_group()


def test_data_parallel_update_on_rank_local_buffers():
    """with rank-local rollout buffers every collected transition is trained on.
    World-2 gloo with DIFFERENT buffers per rank equals one process stepping on the union
    of the two ranks' minibatch shards (global advantage normalisation)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_sharded, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    p0, p1, trained = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    np.testing.assert_array_equal(p0, p1)
    assert trained == 2 * 96 * 2  # both buffers, both epochs
    b, model, st = _bundle()
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=64, sgd_epochs=2)
    opt = torch.optim.Adam(b.parameters(), lr=1e-3)
    bufs = [_buffer(96, model, st.T, seed=10 + r) for r in range(2)]
    adv = torch.cat([x["advantages"] for x in bufs])
    mean, std = adv.mean(), adv.std(correction=0)
    gen = torch.Generator().manual_seed(3)
    for _ in range(cfg.sgd_epochs):
        perm = torch.randperm(96, generator=gen)
        for s0 in range(0, 96, 32):
            sel = perm[s0:s0 + 32]
            batch = {"obs": torch.cat([x["obs"][sel] for x in bufs]),
                     "actions": torch.cat([x["actions"][sel] for x in bufs]),
                     "old_log_probs": torch.cat([x["log_probs"][sel] for x in bufs]),
                     "advantages": (torch.cat([x["advantages"][sel] for x in bufs]) - mean) / (std + 1e-8),
                     "returns": torch.cat([x["returns"][sel] for x in bufs])}
            ppo.minibatch_step(b, opt, batch, cfg)
    ref = torch.cat([p.detach().reshape(-1) for p in b.parameters()]).numpy()
    np.testing.assert_allclose(p0, ref, rtol=2e-5, atol=2e-6)


def test_grad_bucket_views_survive_zero_grad():
    """The reducer's bucket views are re-bound after optimizer.zero_grad(set_to_none=True)."""
    b, model, st = _bundle()
    red = ppo.GradAllReduce(b.parameters())
    opt = torch.optim.Adam(b.parameters(), lr=1e-3)
    red.zero_()
    assert all(p.grad is v for p, v in zip(red.params, red.views))
    opt.zero_grad()
    assert all(p.grad is None for p in red.params)
    red.bind()
    out = b.critic(torch.randn(4, 13)).sum()
    out.backward()
    assert all(p.grad is v for p, v in zip(red.params, red.views))
    assert float(red.flat[:red.n].abs().sum()) > 0.0


def test_ac_mpc_bundle_sizes_match_reference_formula():
    """Actor head T*2*n_z and the flat bucket size quoted in SURVEY.md §8(e)."""
    model = DynModel.quadrotor(dt=0.05)
    st = SolveSettings(T=10, u_min=0.0, u_max=5.886)
    b = PolicyBundle("ac_mpc", 11, model, st, CostHeadScaling.for_model(model, 13))
    assert b.actor.net[-1].out_features == 10 * 2 * 17
    n = sum(p.numel() for p in b.parameters())
    assert n == (11 * 512 + 512 + 512 * 512 + 512 + 512 * 340 + 340) + (11 * 512 + 512 + 512 * 512 + 512 + 513) + 4


@pytest.mark.gpu
def test_ac_mpc_minibatch_step_on_gpu():
    from paper_2605_29155_b200 import problems
    from paper_2605_29155_b200.layer import MpcSolver, mpc_control

    dev = torch.device("cuda")
    model = DynModel.quadrotor(dt=0.05)
    pb = problems.hover_problem(model, 256, 10, seed=4)
    b, _, _ = _bundle("ac_mpc")
    b = PolicyBundle("ac_mpc", 13, model, pb.settings, CostHeadScaling.for_model(model, 13), hidden=(64, 64)).to(dev)
    solver = MpcSolver(model, pb.settings, device=dev)
    obs = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    x_init = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    U_warm = torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)
    with torch.no_grad():
        u_mean = mpc_control(b, obs, solver, x_init, U_warm)
        sig = torch.exp(b.log_sigma)
        actions = u_mean + sig * torch.randn_like(u_mean)
        lp = torch.distributions.Normal(u_mean, sig).log_prob(actions).sum(-1)
    batch = {"obs": obs, "actions": actions, "old_log_probs": lp, "advantages": torch.randn(256, device=dev),
             "returns": torch.randn(256, device=dev), "x_init": x_init, "U_warm": U_warm}
    cfg = ppo.TrainConfig()
    loss, metrics = ppo.ppo_losses(b, batch, cfg, solver)
    assert abs(float(metrics["mean_ratio"]) - 1.0) < 1e-6  # exact re-solve: ratio 1
    opt = torch.optim.Adam(b.parameters(), lr=1e-4)
    before = [p.detach().clone() for p in b.actor.parameters()]
    loss, _ = ppo.minibatch_step(b, opt, batch, cfg, solver, reducer=ppo.GradAllReduce(b.parameters()))
    assert loss is not None and torch.isfinite(loss)
    moved = sum(float((p.detach() - q).abs().sum()) for p, q in zip(b.actor.parameters(), before))
    assert moved > 0.0  # the cost actor is trained through the DiffMPC layer


@pytest.mark.gpu
def test_device_rollout_collect_and_update():
    """§8(f) row 2: device-resident collection on the batched race env, then a PPO update
    whose first minibatch re-solve reproduces the rollout controls (ratio 1)."""
    from paper_2605_29155_b200 import raceenv
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.rollout import DeviceRollout

    dev = torch.device("cuda")
    model = DynModel.planar_quadrotor(dt=0.05)
    st = SolveSettings(T=5, u_min=0.0, u_max=2 * 0.5 * 9.81)
    torch.manual_seed(0)
    b = PolicyBundle("ac_mpc", raceenv.OBS_DIM, model, st, CostHeadScaling.for_model(model, 6),
                     hidden=(64, 64)).to(dev)
    env = raceenv.BatchedRaceEnv(raceenv.hairpin5(), model, 128, device=dev, seed=1)
    solver = MpcSolver(model, st, device=dev)
    cfg = ppo.TrainConfig(steps_per_update=6, minibatch_size=256, sgd_epochs=1)
    col = DeviceRollout(b, solver, env, cfg, seed=2)
    flat, stats = col.collect()
    assert flat["obs"].shape == (6 * 128, raceenv.OBS_DIM) and flat["U_warm"].shape == (6 * 128, 5, 2)
    for k, v in flat.items():
        assert bool(torch.isfinite(v).all()), k
    batch = {"obs": flat["obs"][:256], "actions": flat["actions"][:256], "old_log_probs": flat["log_probs"][:256],
             "advantages": flat["advantages"][:256].float(), "returns": flat["returns"][:256].float(),
             "x_init": flat["x_init"][:256], "U_warm": flat["U_warm"][:256]}
    _, metrics = ppo.ppo_losses(b, batch, cfg, solver)
    # the re-solve of a rollout sample reproduces its control bit for bit (trainer.py:9-12)
    assert float(metrics["mean_ratio"]) == 1.0
    opt = torch.optim.Adam(b.parameters(), lr=1e-4)
    out = ppo.ppo_update(flat, b, opt, cfg, solver, generator=torch.Generator().manual_seed(0))
    assert out["skipped_minibatches"] == 0
    assert int(stats["solves"]) == 6 * 128


@pytest.mark.gpu
def test_graphed_minibatch_step_matches_eager():
    """ppo.GraphedMinibatchStep (losses + backward through the DiffMPC layer + clipping
    replayed from one CUDA graph, optimizer step eager) updates the parameters exactly like
    the eager minibatch_step on the same batches."""
    import copy

    from paper_2605_29155_b200 import DynModel, ppo, problems
    from paper_2605_29155_b200.layer import MpcSolver, mpc_control
    from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle

    dev = torch.device("cuda")
    model = DynModel.quadrotor(dt=0.05)
    B, T = 256, 10
    pb = problems.hover_problem(model, B, T, seed=3)
    torch.manual_seed(0)
    b1 = PolicyBundle("ac_mpc", 13, model, pb.settings, CostHeadScaling.for_model(model, 13)).to(dev)
    b2 = copy.deepcopy(b1)
    solver = MpcSolver(model, pb.settings, device=dev)
    cfg = ppo.TrainConfig()
    o1 = torch.optim.Adam(b1.parameters(), lr=cfg.lr_start)
    o2 = torch.optim.Adam(b2.parameters(), lr=cfg.lr_start)
    x_init = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    U_warm = torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)
    g = torch.Generator(device=dev).manual_seed(5)

    def make_batch():
        with torch.no_grad():
            u = mpc_control(b1, x_init, solver, x_init, U_warm)
            sig = torch.exp(b1.log_sigma)
            a = u + sig * torch.randn(u.shape, device=dev, generator=g)
            lp = torch.distributions.Normal(u, sig).log_prob(a).sum(-1)
        return {"obs": x_init.clone(), "actions": a, "old_log_probs": lp,
                "advantages": torch.randn(B, device=dev, generator=g),
                "returns": torch.randn(B, device=dev, generator=g), "x_init": x_init, "U_warm": U_warm}

    batches = [make_batch() for _ in range(4)]
    gstep = ppo.GraphedMinibatchStep(b2, o2, batches[0], cfg, solver)
    assert gstep.diffmpc_launches == 2
    for bt in batches:
        l1, _ = ppo.minibatch_step(b1, o1, bt, cfg, solver)
        l2 = gstep(bt)
        torch.testing.assert_close(l2, l1, rtol=1e-5, atol=1e-6)
    for p1, p2 in zip(b1.parameters(), b2.parameters()):
        torch.testing.assert_close(p2, p1, rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_ppo_update_with_graphed_step_matches_eager():
    """ppo_update with a GraphedMinibatchStep gives the same parameters and statistics as the
    eager update over the same buffer (same permutation generator)."""
    import copy

    from paper_2605_29155_b200 import DynModel, ppo, problems

    dev = torch.device("cuda")
    model = DynModel.quadrotor(dt=0.05)
    n, T = 512, 10
    pb = problems.hover_problem(model, n, T, seed=4)
    torch.manual_seed(0)
    from paper_2605_29155_b200.layer import MpcSolver
    b1 = PolicyBundle("ac_mpc", 13, model, pb.settings, CostHeadScaling.for_model(model, 13)).to(dev)
    b2 = copy.deepcopy(b1)
    solver = MpcSolver(model, pb.settings, device=dev)
    cfg = ppo.TrainConfig(minibatch_size=128, sgd_epochs=2)
    o1 = torch.optim.Adam(b1.parameters(), lr=cfg.lr_start)
    o2 = torch.optim.Adam(b2.parameters(), lr=cfg.lr_start)
    g = torch.Generator(device=dev).manual_seed(9)
    x = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    buf = {"obs": x, "actions": torch.randn((n, 4), device=dev, generator=g),
           "log_probs": torch.randn(n, device=dev, generator=g) - 3.0,
           "advantages": torch.randn(n, device=dev, generator=g, dtype=torch.float64),
           "returns": torch.randn(n, device=dev, generator=g, dtype=torch.float64),
           "x_init": x, "U_warm": torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)}
    m1 = ppo.ppo_update(buf, b1, o1, cfg, solver, generator=torch.Generator().manual_seed(2))
    ex = {"obs": x[:128], "actions": buf["actions"][:128], "old_log_probs": buf["log_probs"][:128],
          "advantages": buf["advantages"][:128].float(), "returns": buf["returns"][:128].float(),
          "x_init": x[:128], "U_warm": buf["U_warm"][:128]}
    gs = ppo.GraphedMinibatchStep(b2, o2, ex, cfg, solver)
    m2 = ppo.ppo_update(buf, b2, o2, cfg, solver, generator=torch.Generator().manual_seed(2), graphed=gs)
    for p1, p2 in zip(b1.parameters(), b2.parameters()):
        torch.testing.assert_close(p2, p1, rtol=1e-5, atol=1e-6)
    assert m1["skipped_minibatches"] == m2["skipped_minibatches"]
    assert abs(m1["approx_grad_frac"] - m2["approx_grad_frac"]) < 1e-12
    assert abs(m1["surrogate"] - m2["surrogate"]) <= 1e-5 * max(1.0, abs(m1["surrogate"]))


@pytest.mark.gpu
def test_graphed_rollout_collection_matches_eager():
    """DeviceRollout.collect_graphed (the whole steps x envs collection replayed from one CUDA
    graph) produces the same transitions, advantages and statistics as eager collect calls
    from the same seeds, collection after collection (carried state and RNG streams)."""
    from paper_2605_29155_b200 import raceenv
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.rollout import DeviceRollout

    dev = torch.device("cuda")
    model = DynModel.planar_quadrotor(dt=0.05)
    st = SolveSettings(T=5, u_min=0.0, u_max=2 * 0.5 * 9.81)
    torch.manual_seed(0)
    b = PolicyBundle("ac_mpc", raceenv.OBS_DIM, model, st, CostHeadScaling.for_model(model, 6),
                     hidden=(64, 64)).to(dev)
    cfg = ppo.TrainConfig(steps_per_update=8, minibatch_size=256, sgd_epochs=1)
    cols = []
    for _ in range(2):
        env = raceenv.BatchedRaceEnv(raceenv.hairpin5(), model, 128, device=dev, seed=1)
        cols.append(DeviceRollout(b, MpcSolver(model, st, device=dev), env, cfg, seed=2))
    eager, graphed = cols
    for it in range(4):
        fa, sa = eager.collect()
        fb, sb = graphed.collect_graphed()
        for k in fa:
            torch.testing.assert_close(fb[k], fa[k], rtol=0, atol=0, msg=f"collection {it}: {k}")
        for k in ("episodes", "return_sum", "laps", "solver_iters"):
            assert float(sb[k]) == float(sa[k]), (it, k)
        fa = {k: v.clone() for k, v in fa.items()}
    assert graphed.step_count == eager.step_count


@pytest.mark.gpu
def test_graphed_update_with_partial_last_minibatch():
    """n % minibatch_size != 0 sends the last minibatch through the eager step,
    whose zero_grad(set_to_none) drops the .grad tensors; the graphed step re-binds its bucket
    views before every replay, so parameters still match the all-eager update."""
    import copy

    from paper_2605_29155_b200 import problems
    from paper_2605_29155_b200.layer import MpcSolver

    dev = torch.device("cuda")
    model = DynModel.quadrotor(dt=0.05)
    n, T, mb = 300, 10, 128
    pb = problems.hover_problem(model, n, T, seed=4)
    torch.manual_seed(0)
    b1 = PolicyBundle("ac_mpc", 13, model, pb.settings, CostHeadScaling.for_model(model, 13),
                      hidden=(64, 64)).to(dev)
    b2 = copy.deepcopy(b1)
    solver = MpcSolver(model, pb.settings, device=dev)
    cfg = ppo.TrainConfig(minibatch_size=mb, sgd_epochs=3)
    o1 = torch.optim.Adam(b1.parameters(), lr=cfg.lr_start)
    o2 = torch.optim.Adam(b2.parameters(), lr=cfg.lr_start)
    g = torch.Generator(device=dev).manual_seed(9)
    x = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    buf = {"obs": x, "actions": torch.randn((n, 4), device=dev, generator=g),
           "log_probs": torch.randn(n, device=dev, generator=g) - 3.0,
           "advantages": torch.randn(n, device=dev, generator=g, dtype=torch.float64),
           "returns": torch.randn(n, device=dev, generator=g, dtype=torch.float64),
           "x_init": x, "U_warm": torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)}
    ppo.ppo_update(buf, b1, o1, cfg, solver, generator=torch.Generator().manual_seed(2))
    ex = {"obs": x[:mb], "actions": buf["actions"][:mb], "old_log_probs": buf["log_probs"][:mb],
          "advantages": buf["advantages"][:mb].float(), "returns": buf["returns"][:mb].float(),
          "x_init": x[:mb], "U_warm": buf["U_warm"][:mb]}
    gs = ppo.GraphedMinibatchStep(b2, o2, ex, cfg, solver)
    ppo.ppo_update(buf, b2, o2, cfg, solver, generator=torch.Generator().manual_seed(2), graphed=gs)
    for p1, p2 in zip(b1.parameters(), b2.parameters()):
        torch.testing.assert_close(p2, p1, rtol=1e-5, atol=1e-6)


@pytest.mark.gpu
def test_nccl_allreduce_captures_into_cuda_graph():
    """The mechanism GraphedMinibatchStep relies on at N>1: an NCCL all-reduce of the flat
    bucket captured in a CUDA graph and replayed (world 1 on the one-GPU box)."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        buf = torch.ones(1024, device=dev)
        dist.all_reduce(buf)  # communicator init outside the capture
        torch.cuda.synchronize()
        gr = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            with torch.cuda.graph(gr):
                buf.mul_(2.0)
                dist.all_reduce(buf)
                buf.add_(1.0)
        torch.cuda.current_stream().wait_stream(side)
        buf.fill_(1.0)
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        assert float(buf[0]) == 15.0  # ((1*2+1)*2+1)*2+1
    finally:
        dist.destroy_process_group()
