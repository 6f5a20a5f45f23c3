"""PPO plumbing pinned to the UNMODIFIED reference (tests/golden/ppo.npz, made by
tests/golden/make_ppo_golden.py from /root/reference/pkg/src/fusedmpc/trainer.py):

  gae          trainer.gae (trainer.py:64-91)
  ppo_losses   loss, metrics and every parameter gradient (trainer.py:124-161), ac_mlp on
               CPU and ac_mpc through the B200 layer (float64 solve) on the GPU
  ppo_update   parameters after the shuffled-minibatch epochs (trainer.py:164-215)
  collect      Trainer._policy_means / collect (trainer.py:256-329): x_init = mpc_state,
               per-slot warm-start shift, reset of done envs, GAE over the buffer
"""

import os

import numpy as np
import pytest
import torch

from paper_2605_29155_b200 import DynModel, SolveSettings, ppo, raceenv
from paper_2605_29155_b200.policy import CostHeadScaling, PolicyBundle

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ppo.npz")


@pytest.fixture(scope="module")
def gd():
    z = np.load(GOLD)
    return {k: z[k] for k in z.files}


PLANAR = DynModel.planar_quadrotor(dt=0.05)
ST3 = SolveSettings(T=3, u_min=0.0, u_max=2 * 0.5 * 9.81)


def bundle(gd, mode, prefix, obs_dim=11, device="cpu"):
    b = PolicyBundle(mode, obs_dim, PLANAR, ST3, CostHeadScaling.for_model(PLANAR, 6), hidden=(32, 32))
    sd = {k[len(prefix) + 3:]: torch.from_numpy(v) for k, v in gd.items() if k.startswith(prefix + "_p_")}
    b.load_state_dict(sd, strict=True)  # the reference's parameter names and shapes
    return b.to(device)


def batch(gd, prefix, device="cpu"):
    p = prefix + "_b_"
    out = {}
    for k, v in gd.items():
        if k.startswith(p):
            t = torch.from_numpy(v)
            out[k[len(p):]] = t.to(device)
    return out


def rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(1.0, np.abs(b).max()))


def test_gae_matches_reference(gd):
    adv, ret = ppo.gae(gd["gae_r"], gd["gae_v"], gd["gae_d"], 0.99, 0.95, gd["gae_lv"])
    np.testing.assert_allclose(adv.numpy(), gd["gae_adv"], rtol=1e-14, atol=1e-14)
    np.testing.assert_allclose(ret.numpy(), gd["gae_ret"], rtol=1e-14, atol=1e-14)


def test_ac_mlp_losses_and_gradients_match_reference(gd):
    b = bundle(gd, "ac_mlp", "mlp0")
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=32, sgd_epochs=2)
    loss, met = ppo.ppo_losses(b, batch(gd, "mlp"), cfg)
    loss.backward()
    assert rel(float(loss.detach()), gd["mlp_loss"]) <= 1e-6
    for k in ("surrogate", "actor_loss", "value_loss", "entropy", "mean_ratio"):
        assert rel(float(met[k]), gd[f"mlp_m_{k}"]) <= 1e-6, k
    for k, p in b.named_parameters():
        assert rel(p.grad.numpy(), gd[f"mlp_g_{k}"]) <= 1e-5, k


def _flat(gd, prefix, device="cpu"):
    f = {}
    for k in ("obs", "actions", "log_probs", "advantages", "returns", "x_init", "U_warm"):
        key = f"{prefix}_{k}"
        if key in gd:
            v = gd[key]
            f[k] = torch.from_numpy(v.reshape(v.shape[0] * v.shape[1], *v.shape[2:])).to(device)
    return f


def test_ac_mlp_update_matches_reference(gd):
    """ppo_update: numpy-style (ddof=0) advantage normalisation, the shared-generator
    permutation, Adam, clipping -> the reference's parameters after 2 epochs."""
    b = bundle(gd, "ac_mlp", "mlp0")
    cfg = ppo.TrainConfig(mode="ac_mlp", minibatch_size=32, sgd_epochs=2)
    opt = torch.optim.Adam(b.parameters(), lr=cfg.lr_start)
    m = ppo.ppo_update(_flat(gd, "mlpu"), b, opt, cfg, generator=torch.Generator().manual_seed(3))
    for k, v in b.state_dict().items():
        assert rel(v.numpy(), gd[f"mlpu_p_{k}"]) <= 1e-5, k
    assert rel(m["surrogate"], gd["mlpu_surrogate"]) <= 1e-5


@pytest.mark.gpu
def test_ac_mpc_losses_and_gradients_match_reference(gd):
    """Through MpcSolveLayer on the GPU (float64 solve + implicit backward kernel)."""
    from paper_2605_29155_b200.layer import MpcSolver

    dev = torch.device("cuda")
    b = bundle(gd, "ac_mpc", "mpc0", device=dev)
    solver = MpcSolver(PLANAR, ST3, device=dev, dtype=torch.float64)
    cfg = ppo.TrainConfig(mode="ac_mpc", minibatch_size=16, sgd_epochs=1)
    bt = batch(gd, "mpc", dev)
    sink = {}
    loss, met = ppo.ppo_losses(b, bt, cfg, solver, sink)
    loss.backward()
    assert int(sink["iterations"]) == int(gd["mpc_iterations"])
    assert rel(float(loss.detach()), gd["mpc_loss"]) <= 1e-5
    for k in ("surrogate", "actor_loss", "value_loss", "entropy", "mean_ratio"):
        assert rel(float(met[k]), gd[f"mpc_m_{k}"]) <= 1e-5, k
    for k, p in b.named_parameters():
        assert rel(p.grad.cpu().numpy(), gd[f"mpc_g_{k}"]) <= 1e-4, k


@pytest.mark.gpu
def test_ac_mpc_update_matches_reference(gd):
    from paper_2605_29155_b200.layer import MpcSolver

    dev = torch.device("cuda")
    b = bundle(gd, "ac_mpc", "mpc0", device=dev)
    solver = MpcSolver(PLANAR, ST3, device=dev, dtype=torch.float64)
    cfg = ppo.TrainConfig(mode="ac_mpc", minibatch_size=16, sgd_epochs=1)
    opt = torch.optim.Adam(b.parameters(), lr=cfg.lr_start)
    m = ppo.ppo_update(_flat(gd, "mpcu", dev), b, opt, cfg, solver, generator=torch.Generator().manual_seed(5))
    for k, v in b.state_dict().items():
        assert rel(v.cpu().numpy(), gd[f"mpcu_p_{k}"]) <= 1e-4, k
    assert rel(m["surrogate"], gd["mpcu_surrogate"]) <= 1e-4


@pytest.mark.gpu
def test_collect_matches_reference(gd):
    """Device-resident collection vs Trainer.collect on the same 6 race envs, weights and
    action noise: x_init = mpc_state (next gate at the origin), the warm start shifted one
    step per env slot, done envs (two time out at step 2) respawned with the default warm
    start, GAE over the buffer."""
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.rollout import DeviceRollout

    dev = torch.device("cuda")
    b = bundle(gd, "ac_mpc", "col0", obs_dim=raceenv.OBS_DIM, device=dev)
    NE = gd["col_x0"].shape[0]
    env = raceenv.BatchedRaceEnv(raceenv.hairpin5(), PLANAR, NE, device=dev, seed=0, reset_noise=0.0)
    solver = MpcSolver(PLANAR, ST3, device=dev, dtype=torch.float64)
    cfg = ppo.TrainConfig(mode="ac_mpc", steps_per_update=gd["col_eps"].shape[0], num_envs=NE)
    col = DeviceRollout(b, solver, env, cfg)  # resets every env to the spawn
    env.x = torch.tensor(gd["col_x0"], dtype=torch.float64, device=dev)
    env.gate = torch.tensor(gd["col_gate0"], dtype=torch.int64, device=dev)
    env.t = torch.tensor(gd["col_t0"], dtype=torch.float64, device=dev)
    col.obs = env.observation().to(torch.float32)
    np.testing.assert_allclose(col.obs.cpu().numpy(), gd["col_obs0"], rtol=1e-6, atol=1e-6)
    eps = torch.tensor(gd["col_eps"], device=dev)
    col.noise = lambda s, shape: eps[s]  # the reference trainer's draws
    flat, stats = col.collect()
    S = gd["col_eps"].shape[0]
    un = lambda k: flat[k].reshape(S, NE, *flat[k].shape[1:]).double().cpu().numpy()  # noqa: E731
    assert np.array_equal(gd["col_dones"].sum(1), np.array([0, 2, 0, 0]))  # the fixture's episode ends
    # step 0 sees identical states; later steps inherit float32-level differences of the
    # actor MLP (cuBLAS vs CPU GEMM) through the executed controls
    assert rel(un("x_init")[0], gd["col_x_init"][0]) <= 1e-12
    for k, tol in (("obs", 1e-5), ("x_init", 1e-5), ("U_warm", 1e-5), ("actions", 1e-5), ("log_probs", 1e-5)):
        assert rel(un(k), gd[f"col_{k}"]) <= tol, k
    assert rel(un("advantages"), gd["col_advantages"]) <= 1e-4
    assert rel(un("returns"), gd["col_returns"]) <= 1e-4
    assert rel(col.warm.cpu().numpy(), gd["col_warm_final"]) <= 1e-5
    assert rel(col.obs.cpu().numpy(), gd["col_obs_final"]) <= 1e-5
    assert int(stats["episodes"]) == int(gd["col_episodes"])


@pytest.mark.gpu
def test_act_matches_reference(gd):
    """policy.act (policy.py:324-366), B = 1 on the GPU in float64: from_diag lift of the
    actor output, one solve warm-started from the slot, push_warm, a Gaussian exploration
    sample (same numpy generator) and its pre-clamp log-density; three consecutive calls."""
    from paper_2605_29155_b200.layer import MpcSolver
    from paper_2605_29155_b200.policy import act

    dev = torch.device("cuda")
    b = bundle(gd, "ac_mpc", "act0", device=dev)
    solver = MpcSolver(PLANAR, ST3, device=dev, dtype=torch.float64, n_slots=2)
    for k in range(gd["act_obs"].shape[0]):
        a = act(b, gd["act_obs"][k], gd["act_x"][k], solver, True, np.random.default_rng(20 + k), slot=1)
        assert rel(a.u_mpc, gd["act_u_mpc"][k]) <= 1e-6
        assert rel(a.u_sampled, gd["act_u_sampled"][k]) <= 1e-6
        assert abs(a.log_prob - gd["act_log_prob"][k]) <= 1e-5 * max(1.0, abs(gd["act_log_prob"][k]))
        assert rel(solver.warm[1].cpu().numpy(), gd["act_warm"][k]) <= 1e-6
