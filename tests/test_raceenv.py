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
