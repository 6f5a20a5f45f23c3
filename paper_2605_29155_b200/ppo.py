"""PPO update with the DiffMPC layer in the actor's gradient path, data-parallel over ranks
(SURVEY.md §8(e) config 4 / §8(f) row 1), mirroring
/root/reference/pkg/src/fusedmpc/trainer.py:37-215 (TrainConfig, gae, ppo_losses,
ppo_update).

Differences from the reference, all on the plumbing side:
  * buffers and minibatches are device tensors; the solver inputs stored by the rollout
    (x_init, U_warm — trainer.py:9-12) stay on the GPU, so a minibatch re-solve
    reproduces the rollout controls exactly and the importance ratio is 1 at the
    trust-region centre (the reference's invariant);
  * with ``torch.distributed`` initialised, every rank holds a full replica and works on
    its own shard of each minibatch; after ``loss.backward()`` the actor + critic +
    log_sigma gradients are flattened into ONE bucket and averaged with a single
    all-reduce (NCCL over NVLink on the B200 box, gloo in the CPU tests), then clipped and
    applied — identical parameters on every rank after every step.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .errors import ConfigError


@dataclass
class TrainConfig:
    """trainer.py:37-63 (same defaults)."""

    gamma: float = 0.99
    lam: float = 0.95
    steps_per_update: int = 256
    minibatch_size: int = 2048
    sgd_epochs: int = 10
    clip_range: float = 0.2
    lr_start: float = 3e-4
    lr_end: float = 3e-5
    entropy_coef: float = 0.0
    value_coef: float = 0.5
    grad_clip: float = 0.5
    total_steps: int = 200_000
    num_envs: int = 16
    mode: str = "ac_mpc"
    normalize_advantages: bool = True
    checkpoint_every: int = 20

    def __post_init__(self):
        if self.mode not in ("ac_mpc", "ac_mlp"):
            raise ConfigError(f"train mode must be ac_mpc or ac_mlp, got {self.mode!r}")
        if not 0.0 <= self.gamma <= 1.0 or not 0.0 <= self.lam <= 1.0:
            raise ConfigError("gamma and lam must lie in [0, 1]")
        if self.steps_per_update < 1 or self.num_envs < 1:
            raise ConfigError("steps_per_update and num_envs must be >= 1")


def gae(rewards, values, dones, gamma, lam, last_values):
    """Generalized advantage estimation over (steps, envs) tensors (trainer.py:66-91).
    Works on any device; accumulation in float64 like the reference."""
    rewards, values, dones, last_values = (torch.as_tensor(a, dtype=torch.float64)
                                           for a in (rewards, values, dones, last_values))
    if not (rewards.shape == values.shape == dones.shape):
        raise ConfigError("rewards, values and dones must share a (steps, envs) shape")
    if tuple(last_values.shape) != tuple(rewards.shape[1:]):
        raise ConfigError("last_values must have one bootstrap entry per env")
    adv = torch.zeros_like(rewards)
    next_adv = torch.zeros_like(last_values)
    next_val = last_values
    for s in range(rewards.shape[0] - 1, -1, -1):
        nonterminal = 1.0 - dones[s]
        delta = rewards[s] + gamma * next_val * nonterminal - values[s]
        next_adv = delta + gamma * lam * nonterminal * next_adv
        adv[s] = next_adv
        next_val = values[s]
    return adv, adv + values


def ppo_losses(bundle, batch, config: TrainConfig, solver=None, stats_sink=None):
    """Clipped-surrogate PPO losses for one minibatch (trainer.py:124-161).

    batch: obs, actions, old_log_probs, advantages, returns (+ x_init, U_warm in ac_mpc
    mode), all tensors on the solver's device.
    """
    from .layer import mpc_control

    obs = batch["obs"]
    if bundle.mode == "ac_mpc":
        u_mean = mpc_control(bundle, obs, solver, batch["x_init"], batch["U_warm"], stats_sink)
    else:
        u_mean = bundle.actor(obs)
    sigma = torch.exp(bundle.log_sigma)
    # no argument validation: it costs a host sync per call (and breaks graph capture); a
    # non-finite mean or sigma gives a non-finite loss, i.e. the skipped minibatch
    dist_ = torch.distributions.Normal(u_mean, sigma, validate_args=False)
    log_probs = dist_.log_prob(batch["actions"]).sum(-1)
    ratio = torch.exp(log_probs - batch["old_log_probs"])
    adv = batch["advantages"]
    surrogate = torch.min(ratio * adv,
                          torch.clamp(ratio, 1.0 - config.clip_range, 1.0 + config.clip_range) * adv).mean()
    actor_loss = -surrogate
    values = bundle.critic(obs)
    value_loss = ((values - batch["returns"]) ** 2).mean()
    entropy = dist_.entropy().sum(-1).mean()
    loss = actor_loss + config.value_coef * value_loss - config.entropy_coef * entropy
    metrics = {"surrogate": surrogate.detach(), "actor_loss": actor_loss.detach(),
               "value_loss": value_loss.detach(), "entropy": entropy.detach(),
               "mean_ratio": ratio.detach().mean()}
    return loss, metrics


class GradAllReduce:
    """One flat gradient bucket per step, averaged over ranks with a single all-reduce.

    The bucket is allocated once (parameter order fixed) and reused; gradients are
    copied in, reduced in place and copied back, so the collective is one launch of
    size sum(numel) (2.85 MB for the T=10, n_z=17 AC-MPC bundle)."""

    def __init__(self, params, group=None):
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        n = sum(p.numel() for p in self.params)
        dev = self.params[0].device
        self.flat = torch.zeros(n, dtype=torch.float32, device=dev)

    @property
    def nbytes(self) -> int:
        return self.flat.numel() * self.flat.element_size()

    def __call__(self):
        if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(self.group) == 1:
            return
        world = dist.get_world_size(self.group)
        off = 0
        for p in self.params:
            n = p.numel()
            if p.grad is None:
                self.flat[off:off + n].zero_()
            else:
                self.flat[off:off + n].copy_(p.grad.reshape(-1))
            off += n
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        self.flat.div_(world)
        off = 0
        for p in self.params:
            n = p.numel()
            g = self.flat[off:off + n].view_as(p)
            if p.grad is None:
                p.grad = g.clone()
            else:
                p.grad.copy_(g)
            off += n


def minibatch_step(bundle, optimizer, batch, config: TrainConfig, solver=None, reducer=None,
                   stats_sink=None):
    """One PPO minibatch step: losses -> backward (through the DiffMPC layer) -> gradient
    all-reduce -> clip -> optimizer step (trainer.py:200-212). Returns (loss, metrics);
    a non-finite loss skips the step on every rank (the reference's skipped minibatch)."""
    loss, metrics = ppo_losses(bundle, batch, config, solver, stats_sink)
    finite = torch.isfinite(loss.detach()).to(torch.float32).reshape(1)
    if reducer is not None and dist.is_available() and dist.is_initialized():
        dist.all_reduce(finite, op=dist.ReduceOp.MIN, group=reducer.group)
    if float(finite.item()) < 1.0:
        return None, metrics
    optimizer.zero_grad()
    loss.backward()
    if reducer is not None:
        reducer()
    torch.nn.utils.clip_grad_norm_([p for p in bundle.parameters() if p.grad is not None], config.grad_clip)
    optimizer.step()
    return loss.detach(), metrics


class GraphedMinibatchStep:
    """minibatch_step with the losses, the backward through the DiffMPC layer and the gradient
    clipping replayed from one CUDA graph (single process, or whenever no collective runs).

    The eager step issues ~130 kernel launches from Python (MLPs, distributions, the solver's
    output allocations, autograd); replaying them as one graph leaves the GPU time. Each call
    copies the minibatch into static buffers, replays the graph, reads the finite-loss flag
    (the reference's skipped minibatch, trainer.py:200-212) and, if finite, runs the
    optimizer step eagerly — the same arithmetic as ``minibatch_step`` on the same batch.
    Warm-up passes (before capture) compute gradients only; parameters are untouched.
    """

    def __init__(self, bundle, optimizer, example_batch: dict, config: TrainConfig, solver=None, warmup: int = 3):
        self.bundle, self.optimizer, self.config, self.solver = bundle, optimizer, config, solver
        self.params = [p for p in bundle.parameters() if p.requires_grad]
        self.static = {k: v.detach().clone() for k, v in example_batch.items()}
        for p in self.params:
            if p.grad is None:
                p.grad = torch.zeros_like(p)
        side = torch.cuda.Stream(device=self.params[0].device)
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            for _ in range(warmup):
                self._body()
        torch.cuda.current_stream().wait_stream(side)
        from . import _lib
        l0 = _lib.launch_count()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph):
            self.loss, self.finite = self._body()
        self.diffmpc_launches = _lib.launch_count() - l0  # DiffMPC kernels inside the graph

    def _body(self):
        for p in self.params:
            p.grad.zero_()
        self.sink = {}  # per-replay solver counters (the tensors written by the graph)
        loss, self.metrics = ppo_losses(self.bundle, self.static, self.config, self.solver, self.sink)
        finite = torch.isfinite(loss.detach())
        loss.backward()
        torch.nn.utils.clip_grad_norm_(self.params, self.config.grad_clip)
        return loss.detach(), finite

    def matches(self, batch: dict) -> bool:
        return all(k in self.static and self.static[k].shape == v.shape for k, v in batch.items())

    def __call__(self, batch: dict, stats_sink=None):
        """One step; returns the loss (a static tensor, valid until the next call) or None for
        a skipped minibatch. ``self.metrics`` holds this step's metrics (static tensors)."""
        for k, v in batch.items():
            self.static[k].copy_(v, non_blocking=True)
        self.graph.replay()
        if stats_sink is not None:
            for k, v in self.sink.items():
                stats_sink[k] = stats_sink.get(k, 0) + v
        if not bool(self.finite.item()):
            return None
        self.optimizer.step()
        return self.loss


def ppo_update(buffer: dict, bundle, optimizer, config: TrainConfig, solver=None, generator=None,
               reducer=None, rank: int = 0, world: int = 1, graphed: GraphedMinibatchStep | None = None):
    """Epochs of shuffled-minibatch updates over a filled buffer (trainer.py:164-215).

    buffer: flat (n, ...) device tensors obs, actions, log_probs, advantages, returns
    (+ x_init, U_warm). Each rank processes its contiguous 1/world slice of every
    minibatch (the permutation is drawn from the shared generator, so all ranks agree).
    ``graphed``: a GraphedMinibatchStep of this bundle/optimizer (one process) replaces the
    eager step for every minibatch of its shape.
    """
    from .shard import shard_range

    n = buffer["obs"].shape[0]
    adv = buffer["advantages"].to(torch.float32)
    if config.normalize_advantages:
        adv = (adv - adv.mean()) / (adv.std() + 1e-8)
    flat = {"obs": buffer["obs"], "actions": buffer["actions"], "old_log_probs": buffer["log_probs"],
            "advantages": adv, "returns": buffer["returns"].to(torch.float32)}
    if bundle.mode == "ac_mpc":
        flat["x_init"] = buffer["x_init"]
        flat["U_warm"] = buffer["U_warm"]
    mb = min(config.minibatch_size, n)
    stats_sink, skipped, last = {}, 0, {}
    for _ in range(config.sgd_epochs):
        perm = torch.randperm(n, generator=generator).to(buffer["obs"].device)
        for start in range(0, n, mb):
            sel = perm[start:start + mb]
            lo, hi = shard_range(sel.shape[0], rank, world)
            sel = sel[lo:hi]
            batch = {k: v[sel] for k, v in flat.items()}
            if graphed is not None and graphed.matches(batch):
                loss = graphed(batch, stats_sink)
                metrics = {k: v.clone() for k, v in graphed.metrics.items()}
            else:
                loss, metrics = minibatch_step(bundle, optimizer, batch, config, solver, reducer, stats_sink)
            if loss is None:
                skipped += 1
                continue
            last = metrics
    solves = stats_sink.get("solves", 0)
    last = {k: float(v) for k, v in last.items()}
    last["skipped_minibatches"] = skipped
    last["approx_grad_frac"] = float(stats_sink.get("non_converged", 0)) / solves if solves else 0.0
    return last
