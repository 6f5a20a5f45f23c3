"""Device-resident rollout collection for AC-MPC PPO, mirroring
Trainer._policy_means / Trainer.collect (/root/reference/pkg/src/fusedmpc/trainer.py:256-329).

Every policy evaluation is one batched forward DiffMPC solve over all environments on the
GPU, warm-started from the previous solution shifted one step (the receding-horizon shift
of policy.py:206-212 / trainer.py:271); the environments (``raceenv.BatchedRaceEnv``),
the warm starts, the solver inputs stored for the minibatch re-solve (x_init, U_warm —
trainer.py:9-12) and the whole (steps, envs) buffer stay in device memory. Nothing is
copied to the host inside the loop; episode statistics are accumulated as device tensors.
"""

from __future__ import annotations

import torch

from .ppo import TrainConfig, gae


class DeviceRollout:
    def __init__(self, bundle, solver, env, config: TrainConfig, seed: int = 0):
        self.bundle, self.solver, self.env, self.config = bundle, solver, env, config
        self.device = env.device
        self.N = env.N
        T, m = bundle.T, bundle.n_u
        self.gen = torch.Generator(device=self.device).manual_seed(seed)
        self.obs = env.reset().to(torch.float32)
        # the solver inputs are kept in the solver's precision (a minibatch re-solve must see
        # exactly what the rollout solve saw; float64 = the reference's precision)
        self.sdt = getattr(solver, "dtype", torch.float32)
        self.default_u = torch.as_tensor(solver.default_u, dtype=self.sdt, device=self.device)
        self.warm = self.default_u.expand(self.N, T, m).clone()
        self.ep_return = torch.zeros(self.N, dtype=torch.float64, device=self.device)
        self.u_lo = torch.as_tensor(bundle.u_min, dtype=torch.float64, device=self.device)
        self.u_hi = torch.as_tensor(bundle.u_max, dtype=torch.float64, device=self.device)
        self.step_count = 0
        self.plan = None

    @torch.no_grad()
    def policy_means(self, obs_t):
        """Control means for all environments (trainer.py:256-274): actor -> batched solve
        -> first control; stores the shifted solution as the next warm start."""
        diag, cvec = self.bundle.actor(obs_t)
        x_init = self.env.mpc_state()
        U_warm = self.warm.clone()
        if self.plan is None:  # preallocated launch (the solve's outputs are consumed here)
            from .solver import SolvePlan
            self.plan = SolvePlan(self.solver.model, self.solver.settings, self.N, layout="diag",
                                  dtype=self.sdt, device=self.device, want_gains=False, backward=False,
                                  kernel=getattr(self.solver, "kernel", "throughput"))
        ws = self.plan.solve(x_init.to(self.sdt).contiguous(), diag.to(self.sdt).contiguous(),
                             cvec.to(self.sdt).contiguous(), U_warm)
        self.warm = torch.cat([ws.U[:, 1:], ws.U[:, -1:]], dim=1)
        return ws.U[:, 0].to(torch.float32, copy=True), x_init, U_warm, ws.iters.clone()  # float32 means (trainer.py:273)

    def noise(self, step, shape):
        """Standard-normal exploration noise of one step (trainer.py:283: one (N, m) draw per
        step from the rollout's generator). Tests substitute the reference's draws."""
        return torch.randn(shape, generator=self.gen, dtype=torch.float32, device=self.device)

    # state carried from one collection to the next (rollout + environment)
    _STATE = ("obs", "warm", "ep_return")
    _ENV_STATE = ("x", "gate", "laps", "t", "done", "reason")

    @torch.no_grad()
    def collect_graphed(self, steps: int | None = None):
        """``collect`` replayed from one CUDA graph holding the whole (steps x envs) loop:
        actor -> batched DiffMPC solve -> critic -> action noise -> environment step, GAE.
        The first call runs ``collect`` eagerly (creating the solver plan) and captures the
        graph; every later call replays it. The carried state (observations, warm starts,
        returns, environment state) lives in fixed buffers that the graph reads at its start
        and writes back at its end; the two RNG streams are registered with the graph, so a
        replay draws fresh noise exactly like an eager call would."""
        S = steps or self.config.steps_per_update
        g = getattr(self, "_graph", None)
        if g is None or self._graph_steps != S:
            out = self.collect(S)  # eager: creates the plan, warms the allocator
            torch.cuda.synchronize(self.device)
            self._static = {k: getattr(self, k).clone() for k in self._STATE}
            self._static_env = {k: getattr(self.env, k).clone() for k in self._ENV_STATE}
            for k, v in self._static.items():
                setattr(self, k, v)
            for k, v in self._static_env.items():
                setattr(self.env, k, v)
            g = torch.cuda.CUDAGraph()
            g.register_generator_state(self.gen)
            g.register_generator_state(self.env.gen)
            side = torch.cuda.Stream(device=self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            steps0 = self.step_count
            from . import _lib
            l0 = _lib.launch_count()
            with torch.cuda.stream(side):
                with torch.cuda.graph(g, stream=side):
                    flat, stats = self.collect(S)
                    for k, v in self._static.items():
                        v.copy_(getattr(self, k))
                    for k, v in self._static_env.items():
                        v.copy_(getattr(self.env, k))
            torch.cuda.current_stream(self.device).wait_stream(side)
            self.step_count = steps0
            for k, v in self._static.items():
                setattr(self, k, v)
            for k, v in self._static_env.items():
                setattr(self.env, k, v)
            self.graph_launches = _lib.launch_count() - l0  # DiffMPC kernels per replay
            self._graph, self._graph_steps, self._graph_out = g, S, (flat, stats)
            return out
        g.replay()
        from . import _lib
        _lib.note_graph_replay(self.graph_launches)
        self.step_count += S * self.N
        return self._graph_out

    @torch.no_grad()
    def collect(self, steps: int | None = None):
        """One buffer of (steps, envs) transitions + GAE (trainer.py:276-329). Returns the
        flat buffer dict consumed by ``ppo.ppo_update`` and device-side statistics."""
        cfg = self.config
        S = steps or cfg.steps_per_update
        N, dev = self.N, self.device
        b = self.bundle
        f32 = dict(dtype=torch.float32, device=dev)
        buf = {"obs": torch.empty((S, N, b.obs_dim), **f32), "actions": torch.empty((S, N, b.n_u), **f32),
               "log_probs": torch.empty((S, N), **f32), "values": torch.empty((S, N), dtype=torch.float64, device=dev),
               "rewards": torch.empty((S, N), dtype=torch.float64, device=dev),
               "dones": torch.empty((S, N), dtype=torch.float64, device=dev),
               "x_init": torch.empty((S, N, b.n_x), dtype=self.sdt, device=dev),
               "U_warm": torch.empty((S, N, b.T, b.n_u), dtype=self.sdt, device=dev)}
        sigma = torch.exp(b.log_sigma.detach())
        ep_sum = torch.zeros((), dtype=torch.float64, device=dev)
        ep_cnt = torch.zeros((), dtype=torch.int64, device=dev)
        laps = torch.zeros((), dtype=torch.int64, device=dev)
        iters = torch.zeros((), dtype=torch.int64, device=dev)
        for s in range(S):
            u_mean, x_init, U_warm, it = self.policy_means(self.obs)
            iters += it.sum()
            values = b.critic(self.obs).to(torch.float64)
            eps = self.noise(s, u_mean.shape)
            actions = u_mean + sigma * eps
            log_probs = torch.distributions.Normal(u_mean, sigma, validate_args=False).log_prob(actions).sum(-1)
            u_exec = torch.clamp(actions.to(torch.float64), self.u_lo, self.u_hi)
            buf["obs"][s] = self.obs
            buf["actions"][s] = actions
            buf["log_probs"][s] = log_probs
            buf["values"][s] = values
            buf["x_init"][s] = x_init.to(self.sdt)
            buf["U_warm"][s] = U_warm
            _, reward, done, reason = self.env.step(u_exec)
            buf["rewards"][s] = reward
            buf["dones"][s] = done.to(torch.float64)
            self.ep_return += reward
            ep_sum += torch.where(done, self.ep_return, 0.0).sum()
            ep_cnt += done.sum()
            laps += (done & (reason == 1)).sum()
            self.ep_return = torch.where(done, 0.0, self.ep_return)
            self.warm = torch.where(done[:, None, None], self.default_u, self.warm)
            self.obs = self.env.reset(done).to(torch.float32)
            self.step_count += N
        last_values = b.critic(self.obs).to(torch.float64)
        adv, ret = gae(buf["rewards"], buf["values"], buf["dones"], cfg.gamma, cfg.lam, last_values)
        n = S * N
        flat = {"obs": buf["obs"].reshape(n, -1), "actions": buf["actions"].reshape(n, -1),
                "log_probs": buf["log_probs"].reshape(n), "advantages": adv.reshape(n),
                "returns": ret.reshape(n), "x_init": buf["x_init"].reshape(n, -1),
                "U_warm": buf["U_warm"].reshape(n, b.T, b.n_u)}
        stats = {"episodes": ep_cnt, "return_sum": ep_sum, "laps": laps, "solver_iters": iters, "solves": S * N}
        return flat, stats
