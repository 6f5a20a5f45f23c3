"""Golden vectors for the PPO plumbing around the layer, generated
by the UNMODIFIED reference (/root/reference/pkg/src/fusedmpc/trainer.py, policy.py,
raceenv.py) in the build container. Run once; ppo.npz is committed (the GPU box never reads
/root/reference).

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/nc python tests/golden/make_ppo_golden.py

Contents (prefixes):
  gae_*      trainer.gae on random (steps, envs) buffers with episode boundaries
  mlp_*      ac_mlp bundle (weights), ppo_losses on one minibatch (loss, metrics, every
             parameter gradient) and ppo_update over a buffer (parameters after 2 epochs)
  mpc_*      ac_mpc planar bundle: ppo_losses through MpcSolveLayer (float64 reference
             solve + implicit backward), its gradients, and ppo_update's parameters
  col_*      Trainer.collect: 4 steps x 6 race envs (ac_mpc), with the action noise the
             trainer drew, two envs timing out at step 2 (warm-start and observation reset)
  act_*      policy.act, the B=1 deployment step: three consecutive exploring calls on one
             solver slot (from_diag lift, solve, push_warm, Gaussian sample, log-prob)
"""
import os

import numpy as np
import torch
from fusedmpc import raceenv, trainer
from fusedmpc.batchexec import WorkerPool
from fusedmpc.dynamics import DynModel
from fusedmpc.ilqr import SolveSettings
from fusedmpc.policy import CostHeadScaling, MpcSolver, PolicyBundle, mpc_control

here = os.path.dirname(os.path.abspath(__file__))
out = {}


def params(b, prefix):
    for k, v in b.state_dict().items():
        out[f"{prefix}_p_{k}"] = v.detach().numpy().copy()


def grads(b, prefix):
    for k, p in b.named_parameters():
        out[f"{prefix}_g_{k}"] = (p.grad if p.grad is not None else torch.zeros_like(p)).numpy().copy()


# ----------------------------------------------------------------------------- gae
rng = np.random.default_rng(0)
S, N = 9, 5
r, v = rng.normal(size=(S, N)), rng.normal(size=(S, N))
d = (rng.random((S, N)) < 0.2).astype(float)
lv = rng.normal(size=N)
adv, ret = trainer.gae(r, v, d, 0.99, 0.95, lv)
out.update(gae_r=r, gae_v=v, gae_d=d, gae_lv=lv, gae_adv=adv, gae_ret=ret)

planar = DynModel.planar_quadrotor(dt=0.05)
st3 = SolveSettings(T=3, u_min=0.0, u_max=2 * 0.5 * 9.81)
scal = CostHeadScaling.for_model(planar, 6)


def batch_for(n, obs_dim, n_u, seed, with_mpc=False, b=None, solver=None):
    g = torch.Generator().manual_seed(seed)
    bt = {"obs": torch.randn(n, obs_dim, generator=g), "advantages": torch.randn(n, generator=g),
          "returns": torch.randn(n, generator=g)}
    if with_mpc:
        x = 0.3 * torch.randn(n, 6, generator=g, dtype=torch.float64).numpy()
        Uw = np.tile(solver.default_u, (n, st3.T, 1))
        bt["x_init"], bt["U_warm"] = x, Uw
        with torch.no_grad():
            u = mpc_control(b, bt["obs"], solver, x, Uw)
    else:
        with torch.no_grad():
            u = b.actor(bt["obs"])
    sig = torch.exp(b.log_sigma.detach())
    a = u + sig * torch.randn(u.shape, generator=g)
    bt["actions"] = a
    bt["old_log_probs"] = torch.distributions.Normal(u, sig).log_prob(a).sum(-1) + 0.05 * torch.randn(n, generator=g)
    return bt


def save_batch(bt, prefix):
    for k, val in bt.items():
        out[f"{prefix}_b_{k}"] = val.numpy() if isinstance(val, torch.Tensor) else np.asarray(val)


# ----------------------------------------------------------------------------- ac_mlp
torch.manual_seed(0)
bm = PolicyBundle("ac_mlp", 11, planar, st3, scal, hidden=(32, 32))
params(bm, "mlp0")
cfg = trainer.TrainConfig(mode="ac_mlp", minibatch_size=32, sgd_epochs=2)
bt = batch_for(48, 11, 2, 1, b=bm)
save_batch(bt, "mlp")
loss, met = trainer.ppo_losses(bm, bt, cfg)
loss.backward()
grads(bm, "mlp")
out["mlp_loss"] = float(loss)
for k, val in met.items():
    out[f"mlp_m_{k}"] = val
bm.zero_grad()
# ppo_update over a (8 steps x 16 envs) buffer
buf = trainer.RolloutBuffer.allocate(8, 16, 11, 6, 2, 3)
g = np.random.default_rng(3)
buf.obs[:] = g.normal(size=buf.obs.shape)
buf.actions[:] = g.uniform(0, 9.81, size=buf.actions.shape)
buf.log_probs[:] = g.normal(size=buf.log_probs.shape) - 3.0
buf.advantages = g.normal(size=(8, 16))
buf.returns = g.normal(size=(8, 16))
for k in ("obs", "actions", "log_probs", "advantages", "returns"):
    out[f"mlpu_{k}"] = getattr(buf, k)
opt = torch.optim.Adam(bm.parameters(), lr=cfg.lr_start)
m = trainer.ppo_update(buf, bm, opt, cfg, None, torch.Generator().manual_seed(3))
params(bm, "mlpu")
out["mlpu_surrogate"] = m["surrogate"]

# ----------------------------------------------------------------------------- ac_mpc
torch.manual_seed(1)
bp = PolicyBundle("ac_mpc", 11, planar, st3, scal, hidden=(32, 32))
params(bp, "mpc0")
solver = MpcSolver(planar, st3, WorkerPool(1))
cfgm = trainer.TrainConfig(mode="ac_mpc", minibatch_size=16, sgd_epochs=1)
bt = batch_for(32, 11, 2, 2, with_mpc=True, b=bp, solver=solver)
save_batch(bt, "mpc")
sink = {}
loss, met = trainer.ppo_losses(bp, bt, cfgm, solver, sink)
loss.backward()
grads(bp, "mpc")
out["mpc_loss"] = float(loss)
for k, val in met.items():
    out[f"mpc_m_{k}"] = val
out["mpc_iterations"] = sink["iterations"]
bp.zero_grad()
buf = trainer.RolloutBuffer.allocate(4, 8, 11, 6, 2, 3)
g = np.random.default_rng(4)
buf.obs[:] = g.normal(size=buf.obs.shape)
buf.actions[:] = g.uniform(0, 9.81, size=buf.actions.shape)
buf.log_probs[:] = g.normal(size=buf.log_probs.shape) - 3.0
buf.advantages = g.normal(size=(4, 8))
buf.returns = g.normal(size=(4, 8))
buf.x_init[:] = 0.3 * g.normal(size=buf.x_init.shape)
buf.U_warm[:] = g.uniform(2.0, 7.0, size=buf.U_warm.shape)
for k in ("obs", "actions", "log_probs", "advantages", "returns", "x_init", "U_warm"):
    out[f"mpcu_{k}"] = getattr(buf, k)
opt = torch.optim.Adam(bp.parameters(), lr=cfgm.lr_start)
m = trainer.ppo_update(buf, bp, opt, cfgm, solver, torch.Generator().manual_seed(5))
params(bp, "mpcu")
out["mpcu_surrogate"] = m["surrogate"]

# ----------------------------------------------------------------------------- collect
torch.manual_seed(2)
bc = PolicyBundle("ac_mpc", raceenv.OBS_DIM, planar, st3, scal, hidden=(32, 32))
params(bc, "col0")
track = raceenv.load_track("/root/reference/pkg/src/fusedmpc/tracks/hairpin5.yaml")
NE = 6
envs = [raceenv.RaceEnv(track, planar, seed=10 + i, reset_noise=0.0) for i in range(NE)]
ccfg = trainer.TrainConfig(mode="ac_mpc", steps_per_update=4, num_envs=NE)
tr = trainer.Trainer(ccfg, bc, envs, MpcSolver(planar, st3, WorkerPool(1), n_slots=NE), "/tmp/ppo_golden_run", seed=7)
g = np.random.default_rng(6)
X0, G0, T0 = [], [], []
for i, env in enumerate(envs):
    gi = int(g.integers(len(track.gates)))
    gate = track.gates[gi]
    p = gate.center - g.uniform(1.0, 3.0) * gate.normal
    x = np.array([p[0], p[1], g.normal(0, 0.1), *(gate.normal * g.uniform(1, 4)), g.normal(0, 0.3)])
    t0 = 19.93 if i in (1, 4) else 3.0
    env.state = raceenv.EnvState(x=x, next_gate_index=gi, episode_time=t0)
    X0.append(x), G0.append(gi), T0.append(t0)
    tr.obs[i] = raceenv.observation(env.state, track).astype(np.float32)
out.update(col_x0=np.array(X0), col_gate0=np.array(G0), col_t0=np.array(T0), col_obs0=tr.obs.copy())
# the action noise the trainer draws (same generator, same order: one (N, m) draw per step)
gen = torch.Generator().manual_seed(7)
out["col_eps"] = np.stack([torch.randn((NE, 2), generator=gen).numpy() for _ in range(ccfg.steps_per_update)])
cb, episodes = tr.collect()
for k in ("obs", "actions", "log_probs", "rewards", "values", "dones", "x_init", "U_warm", "advantages", "returns"):
    out[f"col_{k}"] = getattr(cb, k)
out["col_warm_final"] = tr.warm.copy()
out["col_obs_final"] = tr.obs.copy()
out["col_episodes"] = len(episodes)

# ----------------------------------------------------------------------------- act (B = 1)
from fusedmpc.policy import act  # noqa: E402

asolver = MpcSolver(planar, st3, WorkerPool(1), n_slots=2)
g = np.random.default_rng(8)
AO, AX, AU, AS, AL, AW = [], [], [], [], [], []
for k in range(3):  # consecutive calls on slot 1: the receding-horizon warm start carries over
    obs = g.normal(size=11)
    x = np.array([0.3, -0.2, 0.05, 0.5, -0.3, 0.1]) + 0.05 * k
    a = act(bp, obs, x, asolver, True, np.random.default_rng(20 + k), slot=1)
    AO.append(obs), AX.append(x), AU.append(a.u_mpc), AS.append(a.u_sampled), AL.append(a.log_prob)
    AW.append(asolver.warm[1].copy())
out.update(act_obs=np.array(AO), act_x=np.array(AX), act_u_mpc=np.array(AU), act_u_sampled=np.array(AS),
           act_log_prob=np.array(AL), act_warm=np.array(AW))
params(bp, "act0")

np.savez_compressed(os.path.join(here, "ppo.npz"), **{k: np.asarray(v) for k, v in out.items()})
print(len(out), "arrays; dones per step", cb.dones.sum(1), "episodes", len(episodes))
