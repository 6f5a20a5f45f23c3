"""Batched GPU race environment against golden vectors from the
reference's own env_step / observation / mpc_state (tests/golden/make_env_golden.py):
gate passes, lap completion, misses, out-of-bounds, timeouts and shaped rewards."""

import os

import numpy as np
import pytest
import torch

from paper_2605_29155_b200 import DynModel
from paper_2605_29155_b200 import raceenv

GOLD = os.path.join(os.path.dirname(__file__), "golden", "raceenv.npz")


def test_track_and_config_host_logic():
    tr = raceenv.hairpin5()
    assert len(tr.gates) == 5 and tr.laps == 1
    np.testing.assert_allclose(tr.lo, [-5.0, -5.0])
    np.testing.assert_allclose(tr.hi, [14.0, 14.0])
    with pytest.raises(Exception):
        raceenv.Gate(np.zeros(2), np.array([1.0, 1.0]), 1.0)


@pytest.mark.gpu
def test_env_step_matches_reference_goldens():
    g = np.load(GOLD)
    N = g["x0"].shape[0]
    env = raceenv.BatchedRaceEnv(raceenv.hairpin5(), DynModel.planar_quadrotor(dt=0.05), N, device="cuda")
    f = dict(dtype=torch.float64, device="cuda")
    env.x = torch.tensor(g["x0"], **f)
    env.gate = torch.tensor(g["gate0"], dtype=torch.int64, device="cuda")
    env.laps = torch.tensor(g["laps0"], dtype=torch.int64, device="cuda")
    env.t = torch.tensor(g["t0"], **f)
    np.testing.assert_allclose(env.observation().cpu().numpy(), g["obs0"], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(env.mpc_state().cpu().numpy(), g["mpc0"], rtol=1e-12, atol=1e-12)
    obs, rew, done, reason = env.step(torch.tensor(g["u"], **f))
    np.testing.assert_array_equal(reason.cpu().numpy(), g["reason"])
    np.testing.assert_array_equal(done.cpu().numpy(), g["done"])
    np.testing.assert_array_equal(env.gate.cpu().numpy(), g["gate"])
    np.testing.assert_array_equal(env.laps.cpu().numpy(), g["laps"])
    np.testing.assert_allclose(env.t.cpu().numpy(), g["t"], rtol=0, atol=1e-12)
    fin = np.isfinite(g["x"]).all(1) & (np.abs(g["x"]) < 1e300).all(1)
    np.testing.assert_allclose(env.x.cpu().numpy()[fin], g["x"][fin], rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(rew.cpu().numpy()[fin], g["reward"][fin], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(obs.cpu().numpy()[fin], g["obs"][fin], rtol=1e-9, atol=1e-9)


@pytest.mark.gpu
def test_done_envs_do_not_advance_and_reset():
    env = raceenv.BatchedRaceEnv(raceenv.hairpin5(), DynModel.planar_quadrotor(dt=0.05), 64, device="cuda",
                                 reset_noise=0.1)
    env.reset()
    env.t[:] = 19.99
    u = torch.full((64, 2), 2.4525, dtype=torch.float64, device="cuda")
    _, _, done, reason = env.step(u)
    assert bool(done.all()) and bool((reason == raceenv.REASON_TIMEOUT).all())
    x_before = env.x.clone()
    _, rew, _, _ = env.step(u)
    assert torch.equal(env.x, x_before) and bool((rew == 0).all())
    obs = env.reset(done)
    assert not bool(env.done.any()) and obs.shape == (64, raceenv.OBS_DIM)


def test_helix5_track_is_3d():
    tr = raceenv.helix5()
    assert tr.dim == 3 and len(tr.gates) == 5 and len(tr.spawn) == 13
    for g in tr.gates:
        assert abs(np.linalg.norm(g.normal) - 1.0) < 1e-12
    assert (tr.lo < tr.spawn[:3]).all() and (tr.spawn[:3] < tr.hi).all()
    with pytest.raises(Exception):  # mixed 2-D / 3-D gates
        raceenv.TrackSpec(gates=[raceenv.Gate(np.zeros(2), np.array([1.0, 0.0]), 1.0),
                                 raceenv.Gate(np.zeros(3), np.array([1.0, 0.0, 0.0]), 1.0)], laps=1,
                          spawn=np.zeros(13))


def _step3d_restated(x, gate, laps, t, u, track, cfg, model):
    """numpy restatement of the 3-D environment step (raceenv.py:174-228 semantics with
    circular gate openings), one environment at a time; dynamics from the oracle."""
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
    import oracle
    xn = oracle.dynamics(model, x, u)[0]
    out = []
    for i in range(x.shape[0]):
        g = track.gates[gate[i]]
        r = -cfg.time_penalty * model.dt
        nxt, lp, reason = gate[i], laps[i], 0
        xi = xn[i].copy()
        if not np.isfinite(xi).all():
            xi = np.where(np.isfinite(xi), xi, 0.0)
            reason, r = 3, r - cfg.crash_penalty
        else:
            pp, pn = x[i, 0:3], xi[0:3]
            r += float(np.clip(cfg.k_p * (np.linalg.norm(pp - g.center) - np.linalg.norm(pn - g.center)),
                               -cfg.progress_cap, cfg.progress_cap))
            sp, sn = float(g.normal @ (pp - g.center)), float(g.normal @ (pn - g.center))
            crossed = sp <= 0.0 and sn > 0.0
            lat = 0.0
            if crossed:
                frac = sp / (sp - sn) if sn != sp else 0.0
                pc = pp + frac * (pn - pp) - g.center
                lat = float(np.linalg.norm(pc - (g.normal @ pc) * g.normal))
            hw = g.width / 2.0
            if crossed and lat <= hw:
                r += cfg.gate_bonus
                nxt += 1
                if nxt == len(track.gates):
                    lp, nxt = lp + 1, 0
                    if lp >= track.laps:
                        reason = 1
            elif crossed and lat <= cfg.miss_factor * hw:
                reason, r = 2, r - cfg.crash_penalty
            elif not ((pn >= track.lo).all() and (pn <= track.hi).all()):
                reason, r = 3, r - cfg.crash_penalty
            if reason == 0 and t[i] + model.dt >= cfg.timeout:
                reason = 4
        out.append((xi, nxt, lp, reason, r))
    return out


@pytest.mark.gpu
def test_3d_env_step_matches_restatement():
    """The 13-state environment (no reference exists): the fused kernel vs a numpy
    restatement of the same rules on states around every gate (passes, misses, out of
    bounds, timeouts, a non-finite state, the last gate completing the lap)."""
    tr = raceenv.helix5()
    model = DynModel.quadrotor(dt=0.05)
    cfg = raceenv.RewardConfig()
    rng = np.random.default_rng(3)
    N = 512
    x = np.zeros((N, 13))
    gate = rng.integers(0, 5, size=N)
    for i in range(N):
        g = tr.gates[gate[i]]
        a = rng.normal(size=3)
        a -= (a @ g.normal) * g.normal
        lat = rng.uniform(0, 2.5) * g.width / 2 * a / np.linalg.norm(a)
        x[i, 0:3] = g.center - rng.uniform(0.0, 0.3) * g.normal + lat
        q = np.array([1.0, 0, 0, 0]) + 0.1 * rng.normal(size=4)
        x[i, 3:7] = q / np.linalg.norm(q)
        x[i, 7:10] = g.normal * rng.uniform(0.0, 10.0) + rng.normal(0, 0.5, size=3)
        x[i, 10:13] = rng.normal(0, 0.5, size=3)
    x[::41, 0:3] = tr.hi + 1.0       # out of bounds
    x[7, 7] = 1e308                   # overflow -> non-finite
    t = rng.choice([0.0, 3.0, 19.97], size=N)
    u = rng.uniform(0.0, 0.6 * 9.81, size=(N, 4))
    env = raceenv.BatchedRaceEnv(tr, model, N, device="cuda")
    f = dict(dtype=torch.float64, device="cuda")
    env.x, env.t = torch.tensor(x, **f), torch.tensor(t, **f)
    env.gate = torch.tensor(gate, dtype=torch.int64, device="cuda")
    from paper_2605_29155_b200 import _lib
    l0 = _lib.launch_count()
    obs, rew, done, reason = env.step(torch.tensor(u, **f))
    assert _lib.launch_count() - l0 == 1  # one fused kernel per step
    ref = _step3d_restated(x, gate, np.zeros(N, np.int64), t, u, tr, cfg, model)
    reasons = np.array([r[3] for r in ref])
    assert set(np.unique(reasons)) >= {0, 2, 3, 4}
    np.testing.assert_array_equal(reason.cpu().numpy(), reasons)
    np.testing.assert_array_equal(env.gate.cpu().numpy(), [r[1] for r in ref])
    np.testing.assert_allclose(env.x.cpu().numpy(), np.array([r[0] for r in ref]), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(rew.cpu().numpy(), [r[4] for r in ref], rtol=1e-9, atol=1e-9)
    np.testing.assert_allclose(obs.cpu().numpy(), env.observation().cpu().numpy(), rtol=1e-12, atol=1e-12)
    assert obs.shape == (N, raceenv.OBS_DIM_3D)
