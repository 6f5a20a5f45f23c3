"""BASELINE config 4: AC-MPC PPO minibatch step with the DiffMPC actor, data-parallel.

    python bench_ppo.py [--steps K --warmup W --minibatch B]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N --master-addr 127.0.0.1 \\
        --master-port P bench_ppo.py --gpus N

One step = one PPO minibatch update on every rank (ppo.minibatch_step): cost actor MLP ->
DiffMPC forward (fused iLQR kernel, diagonal cost, T=10, 13-state quadrotor) -> clipped
surrogate + value loss -> backward through the implicit DiffMPC backward kernel -> actor /
critic MLP backward -> ONE flat NCCL all-reduce of the 712,537 gradients -> clip -> Adam.
Each rank owns a B-sample shard (weak scaling). Synthetic rollout data (random-init
networks, hover-problem states as x_init, the rollout controls re-solved exactly so the
importance ratio is 1). Prints one JSON line on rank 0; timings are CUDA events, max over
ranks.
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--minibatch", type=int, default=2048, help="samples per rank per step")
    ap.add_argument("--T", type=int, default=10)
    ap.add_argument("--mode", default="update", choices=["update", "train"],
                    help="update: PPO minibatch steps (13-state quadrotor); train: full device-resident "
                         "PPO iterations (batched race env rollout collection + update)")
    ap.add_argument("--envs", type=int, default=1024, help="train mode: environments per GPU")
    ap.add_argument("--model", default="quad13", choices=["quad13", "planar"],
                    help="train mode: 13-state quadrotor on the 3-D helix5 track (BASELINE model) or the "
                         "reference's planar quadrotor on hairpin5")
    ap.add_argument("--rollout-steps", type=int, default=32, help="train mode: steps per update")
    ap.add_argument("--no-graph", action="store_true",
                    help="update mode: eager minibatch steps (default: one CUDA graph per step when "
                         "no gradient collective runs, i.e. one process)")
    args = ap.parse_args()
    if args.mode == "train":
        return train_mode(args)

    import torch
    import torch.distributed as dist

    from paper_2605_29155_b200 import DynModel, _lib, ppo, problems
    from paper_2605_29155_b200.layer import MpcSolver, mpc_control
    from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DIFFMPC_DRYRUN_SHARE_GPU=1: every rank on cuda:0 over gloo (exercises the multi-rank
    # path on a one-GPU box; never used for reported numbers)
    share = os.environ.get("DIFFMPC_DRYRUN_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl", **({} if share else {"device_id": dev}))
    B, T = args.minibatch, args.T
    model = DynModel.quadrotor(dt=0.05)
    pb = problems.hover_problem(model, B, T, seed=100 + rank)
    torch.manual_seed(0)  # identical replicas on every rank
    obs_dim = 13
    bundle = PolicyBundle("ac_mpc", obs_dim, model, pb.settings, CostHeadScaling.for_model(model, 13)).to(dev)
    solver = MpcSolver(model, pb.settings, device=dev)
    cfg = ppo.TrainConfig()
    opt = torch.optim.Adam(bundle.parameters(), lr=cfg.lr_start)
    reducer = ppo.GradAllReduce(bundle.parameters())
    x_init = torch.tensor(pb.x0, dtype=torch.float32, device=dev)
    U_warm = torch.tensor(pb.U_warm, dtype=torch.float32, device=dev)
    obs = x_init.clone()
    g = torch.Generator(device=dev).manual_seed(1 + rank)
    with torch.no_grad():
        u_mean = mpc_control(bundle, obs, solver, x_init, U_warm)
        sig = torch.exp(bundle.log_sigma)
        actions = u_mean + sig * torch.randn(u_mean.shape, device=dev, generator=g)
        lp = torch.distributions.Normal(u_mean, sig).log_prob(actions).sum(-1)
    batch = {"obs": obs, "actions": actions, "old_log_probs": lp,
             "advantages": torch.randn(B, device=dev, generator=g), "returns": torch.randn(B, device=dev, generator=g),
             "x_init": x_init, "U_warm": U_warm}
    sink = {}
    use_graph = not args.no_graph  # NCCL all-reduce captured in the graph; gloo dry-run reduces eagerly
    if use_graph:
        gstep = ppo.GraphedMinibatchStep(bundle, opt, batch, cfg, solver, reducer=reducer)

        def step(sink_):
            gstep(batch, sink_)
    else:
        def step(sink_):
            ppo.minibatch_step(bundle, opt, batch, cfg, solver, reducer, sink_)
    for _ in range(args.warmup):
        step(sink)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = _lib.launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    sink = {}
    a.record()
    for _ in range(args.steps):
        step(sink)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    launches = (_lib.launch_count() - l0) / args.steps  # graph replays included (_lib.note_graph_replay)
    if rank == 0:
        print(json.dumps({
            "metric": "AC-MPC PPO minibatch steps/s (DiffMPC actor fwd+bwd + grad all-reduce at N>1)",
            "value": 1e3 / ms, "unit": "steps/s", "samples_per_s": world * B * 1e3 / ms,
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "weak", "dtype": "f32", "data": "synthetic",
            "config": {"workload": "AC-MPC PPO step, quadrotor13 diag cost", "T": T, "minibatch_per_gpu": B,
                       "global_minibatch": B * world, "params": sum(p.numel() for p in bundle.parameters()),
                       "allreduce_bytes": reducer.nbytes if world > 1 else 0,
                       "collective": (f"one flat all-reduce per step ({dist.get_backend()})" if world > 1
                                      else "none (one process)"),
                       "parallelism": f"dp{world}"},
            "diffmpc_launches_per_step": launches,
            "cuda_graph": use_graph,
            "allreduce_in_graph": bool(use_graph and world > 1 and gstep.in_graph),
            "mean_solver_iters": (float(sink.get("iterations", 0)) / max(1, sink.get("solves", 1))) if sink else None,
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


def train_mode(args):
    """Full PPO iterations on the device: collect (envs x rollout-steps) transitions with
    one batched DiffMPC forward per step on the GPU race environments, GAE, then one epoch
    of minibatch updates (DiffMPC forward + backward per minibatch, one NCCL all-reduce)."""
    import torch
    import torch.distributed as dist

    from paper_2605_29155_b200 import DynModel, SolveSettings, _lib, ppo, raceenv
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle
    from paper_2605_29155_b200.rollout import DeviceRollout

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # DIFFMPC_DRYRUN_SHARE_GPU=1: every rank on cuda:0 over gloo (exercises the multi-rank
    # path on a one-GPU box; never used for reported numbers)
    share = os.environ.get("DIFFMPC_DRYRUN_SHARE_GPU") == "1"
    local = 0 if share else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("gloo" if share else "nccl", **({} if share else {"device_id": dev}))
    if args.model == "quad13":
        model = DynModel.quadrotor(dt=0.05)
        st = SolveSettings(T=args.T, u_min=0.0, u_max=float(model.mass * model.gravity))
        track, obs_dim = raceenv.helix5(), raceenv.OBS_DIM_3D
    else:
        model = DynModel.planar_quadrotor(dt=0.05)
        st = SolveSettings(T=args.T, u_min=0.0, u_max=2 * 0.5 * 9.81)
        track, obs_dim = raceenv.hairpin5(), raceenv.OBS_DIM
    torch.manual_seed(0)
    bundle = PolicyBundle("ac_mpc", obs_dim, model, st, CostHeadScaling.for_model(model, model.n_x)).to(dev)
    env = raceenv.BatchedRaceEnv(track, model, args.envs, device=dev, seed=11 + rank)
    solver = MpcSolver(model, st, device=dev)
    cfg = ppo.TrainConfig(steps_per_update=args.rollout_steps, minibatch_size=args.minibatch, sgd_epochs=1)
    opt = torch.optim.Adam(bundle.parameters(), lr=cfg.lr_start)
    reducer = ppo.GradAllReduce(bundle.parameters())
    col = DeviceRollout(bundle, solver, env, cfg, seed=5 + rank)
    gen = torch.Generator().manual_seed(3)

    graphed = []

    graph_collect = not args.no_graph  # the collection has no collective: graphed at any N
    use_graph = not args.no_graph  # the update graph carries the NCCL all-reduce at N>1

    def iteration():
        flat, stats = col.collect_graphed() if graph_collect else col.collect()
        if not graphed and use_graph:
            # rank-local buffers: each rank trains on all of its own transitions in
            # minibatches of minibatch/world samples (ppo_update data="sharded")
            mb = max(1, min(cfg.minibatch_size, flat["obs"].shape[0] * world) // world)
            ex = {"obs": flat["obs"][:mb], "actions": flat["actions"][:mb], "old_log_probs": flat["log_probs"][:mb],
                  "advantages": flat["advantages"][:mb].float(), "returns": flat["returns"][:mb].float(),
                  "x_init": flat["x_init"][:mb], "U_warm": flat["U_warm"][:mb]}
            graphed.append(ppo.GraphedMinibatchStep(bundle, opt, ex, cfg, solver, reducer=reducer))
        m = ppo.ppo_update(flat, bundle, opt, cfg, solver, generator=gen, reducer=reducer, rank=rank, world=world,
                           graphed=graphed[0] if graphed else None, data="sharded")
        return stats, m

    for _ in range(max(1, args.warmup // 3)):
        iteration()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    l0 = _lib.launch_count()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = max(2, args.steps // 10)
    a.record()
    trained = 0
    for _ in range(K):
        stats, m = iteration()
        trained += m["samples_trained"]
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / K
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    if rank == 0:
        samples = args.envs * args.rollout_steps
        print(json.dumps({
            "metric": f"AC-MPC PPO iterations/s (device-resident rollout + update, {args.model} race env)",
            "value": 1e3 / ms, "unit": "iterations/s", "env_steps_per_s": world * samples * 1e3 / ms,
            "n_gpus": world, "iterations": K, "ms_per_iteration": ms, "higher_is_better": True,
            "scaling": "weak", "dtype": "f32", "data": "synthetic (race env, random-init policy)",
            "config": {"workload": "PPO: collect envs x steps with one DiffMPC forward and one fused env-step "
                                   "kernel per step, GAE, 1 epoch of minibatch updates", "model": args.model,
                       "track": "helix5 (3-D)" if args.model == "quad13" else "hairpin5", "T": args.T,
                       "envs_per_gpu": args.envs,
                       "rollout_steps": args.rollout_steps, "minibatch_per_gpu": args.minibatch // world,
                       "parallelism": f"dp{world}"},
            "diffmpc_launches_per_iteration": (_lib.launch_count() - l0) / K,
            "cuda_graphs": {"collection": graph_collect, "minibatch_update": bool(graphed)},
            "samples_trained_per_iteration": trained / K,
            "mean_solver_iters": float(stats["solver_iters"]) / stats["solves"],
            "episodes_last_iteration": int(stats["episodes"]),
        }), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
