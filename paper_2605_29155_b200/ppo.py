"""PPO update with the DiffMPC layer in the actor's gradient path, data-parallel over ranks
(SURVEY.md §8(e) config 4 / §8(f) row 1), mirroring
/root/reference/pkg/src/fusedmpc/trainer.py:37-215 (TrainConfig, gae, ppo_losses,
ppo_update).

Differences from the reference, all on the plumbing side:
  * buffers and minibatches are device tensors; the solver inputs stored by the rollout
    (x_init, U_warm — trainer.py:9-12) stay on the GPU, so a minibatch re-solve
    reproduces the rollout controls exactly and the importance ratio is 1 at the
    trust-region centre (the reference's invariant);
  * with ``torch.distributed`` initialised, every rank holds a full replica of the
    networks and works on its shard of each global minibatch (replicated buffers: a slice
    of every minibatch; rank-local buffers: minibatch/world samples of its own buffer);
    the actor + critic + log_sigma gradients accumulate into ONE flat bucket and are
    averaged with a single all-reduce (NCCL over NVLink on the B200 box — captured in the
    minibatch CUDA graph — gloo in the CPU tests), then clipped and applied: identical
    parameters on every rank after every step.
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

    The bucket [gradients | finite flag] is allocated once (parameter order fixed) and
    every parameter's ``.grad`` is bound to a view of it (``bind``): autograd accumulates
    into the views in place, so the collective runs on the bucket with no gather/scatter
    copies (2.85 MB + 4 bytes for the T=10, n_z=17 AC-MPC bundle, ONE launch). The flag
    slot carries each rank's "loss is finite" bit through the same all-reduce, so the
    skipped-minibatch decision (trainer.py:200-203) needs no second collective. On NCCL
    the reduction is capturable into the minibatch CUDA graph (GraphedMinibatchStep)."""

    def __init__(self, params, group=None):
        self.params = [p for p in params if p.requires_grad]
        self.group = group
        if any(p.dtype != torch.float32 for p in self.params):
            raise ConfigError("GradAllReduce buckets float32 parameters")
        self.n = sum(p.numel() for p in self.params)
        dev = self.params[0].device
        self.flat = torch.zeros(self.n + 1, dtype=torch.float32, device=dev)
        self.views, off = [], 0
        for p in self.params:
            self.views.append(self.flat[off:off + p.numel()].view_as(p))
            off += p.numel()
        self.flag = self.flat[self.n:]

    @property
    def nbytes(self) -> int:
        """Gradient payload of the all-reduce (the flag adds 4 bytes)."""
        return self.n * self.flat.element_size()

    def world(self) -> int:
        if not (dist.is_available() and dist.is_initialized()):
            return 1
        return dist.get_world_size(self.group)

    def active(self) -> bool:
        return self.world() > 1

    def capturable(self) -> bool:
        """NCCL collectives can be captured into a CUDA graph; gloo (CPU tests) cannot."""
        return self.active() and dist.get_backend(self.group) == "nccl"

    def bind(self):
        """(Re)bind every parameter's .grad to its bucket view. ``optimizer.zero_grad()``
        (set_to_none) or foreign code may have replaced them; a captured graph writes
        into the views, so they must be the tensors the optimizer reads."""
        for p, v in zip(self.params, self.views):
            if p.grad is not v:
                p.grad = v

    def zero_(self):
        self.bind()
        self.flat.zero_()

    def reduce_(self):
        """Sum the bucket over ranks in place; gradients become the rank mean and the flag
        the number of ranks whose loss was finite."""
        w = self.world()
        if w == 1:
            return
        dist.all_reduce(self.flat, op=dist.ReduceOp.SUM, group=self.group)
        self.flat[:self.n].div_(w)


def minibatch_step(bundle, optimizer, batch, config: TrainConfig, solver=None, reducer=None,
                   stats_sink=None):
    """One PPO minibatch step: losses -> backward (through the DiffMPC layer) -> gradient
    all-reduce -> clip -> optimizer step (trainer.py:200-212). Returns (loss, metrics);
    a non-finite loss on any rank skips the step on every rank (the reference's skipped
    minibatch, decided through the flag slot of the same all-reduce)."""
    loss, metrics = ppo_losses(bundle, batch, config, solver, stats_sink)
    if reducer is None:
        if not bool(torch.isfinite(loss.detach())):
            return None, metrics
        optimizer.zero_grad()
        loss.backward()
        params = [p for p in bundle.parameters() if p.grad is not None]
    else:
        reducer.zero_()
        loss.backward()
        reducer.flag.copy_(torch.isfinite(loss.detach()).reshape(1))
        reducer.reduce_()
        if float(reducer.flag.item()) < reducer.world():
            return None, metrics
        params = reducer.params
    torch.nn.utils.clip_grad_norm_(params, config.grad_clip)
    optimizer.step()
    return loss.detach(), metrics


class GraphedMinibatchStep:
    """minibatch_step with the losses, the backward through the DiffMPC layer, the gradient
    all-reduce (NCCL) and the clipping replayed from one CUDA graph.

    The eager step issues ~130 kernel launches from Python (MLPs, distributions, the solver's
    output allocations, autograd); replaying them as one graph leaves the GPU time. Each call
    copies the minibatch into static buffers, replays the graph, reads the finite-loss flag
    (the reference's skipped minibatch, trainer.py:200-212; summed over ranks by the same
    all-reduce) and, if every rank's loss is finite, runs the optimizer step eagerly — the
    same arithmetic as ``minibatch_step`` on the same batch. Gradients live in the reducer's
    flat bucket (bound as the parameters' ``.grad`` before every replay). A collective that
    cannot be captured (gloo) runs eagerly between the replay and the clipping.
    Warm-up passes (before capture) compute gradients only; parameters are untouched.
    """

    def __init__(self, bundle, optimizer, example_batch: dict, config: TrainConfig, solver=None, warmup: int = 3,
                 reducer: GradAllReduce | None = None):
        self.bundle, self.optimizer, self.config, self.solver = bundle, optimizer, config, solver
        self.reducer = reducer if reducer is not None else GradAllReduce(bundle.parameters())
        self.params = self.reducer.params
        self.in_graph = self.reducer.capturable() or not self.reducer.active()  # collective captured
        self.static = {k: v.detach().clone() for k, v in example_batch.items()}
        self.reducer.bind()
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
            self.loss = self._body()
        self.diffmpc_launches = _lib.launch_count() - l0  # DiffMPC kernels inside the graph

    def _body(self):
        self.reducer.flat.zero_()
        self.sink = {}  # per-replay solver counters (the tensors written by the graph)
        loss, self.metrics = ppo_losses(self.bundle, self.static, self.config, self.solver, self.sink)
        loss.backward()
        self.reducer.flag.copy_(torch.isfinite(loss.detach()).reshape(1))
        if self.in_graph:
            self.reducer.reduce_()
            torch.nn.utils.clip_grad_norm_(self.params, self.config.grad_clip)
        return loss.detach()

    def matches(self, batch: dict) -> bool:
        return all(k in self.static and self.static[k].shape == v.shape for k, v in batch.items())

    def __call__(self, batch: dict, stats_sink=None):
        """One step; returns the loss (a static tensor, valid until the next call) or None for
        a skipped minibatch. ``self.metrics`` holds this step's metrics (static tensors)."""
        for k, v in batch.items():
            self.static[k].copy_(v, non_blocking=True)
        self.reducer.bind()  # an eager step in between may have replaced the .grad tensors
        self.graph.replay()
        from . import _lib
        _lib.note_graph_replay(self.diffmpc_launches)
        if not self.in_graph:
            self.reducer.reduce_()
            torch.nn.utils.clip_grad_norm_(self.params, self.config.grad_clip)
        if stats_sink is not None:
            for k, v in self.sink.items():
                stats_sink[k] = stats_sink.get(k, 0) + v
        if float(self.reducer.flag.item()) < self.reducer.world():
            return None
        self.optimizer.step()
        return self.loss


def ppo_update(buffer: dict, bundle, optimizer, config: TrainConfig, solver=None, generator=None,
               reducer=None, rank: int = 0, world: int = 1, graphed: GraphedMinibatchStep | None = None,
               data: str = "replicated"):
    """Epochs of shuffled-minibatch updates over a filled buffer (trainer.py:164-215).

    buffer: flat (n, ...) device tensors obs, actions, log_probs, advantages, returns
    (+ x_init, U_warm). With ``world`` > 1 the global minibatch of ``config.minibatch_size``
    samples is split over the ranks, in one of two data layouts:
      * ``data="replicated"``: every rank holds the SAME buffer; the permutation is drawn
        from the shared generator (all ranks agree) and each rank takes its contiguous
        1/world slice of every minibatch;
      * ``data="sharded"``: every rank holds its OWN buffer (its environments' transitions,
        equal sizes on all ranks); each rank permutes its whole local buffer and takes
        minibatches of minibatch_size/world samples from it, so every collected transition
        is trained on and the global minibatch is the union of the ranks' shards.
    Advantage normalisation uses the statistics of the whole (global) buffer in both layouts.
    ``graphed``: a GraphedMinibatchStep of this bundle/optimizer replaces the eager step for
    every minibatch of its shape.
    """
    from .shard import shard_range

    if data not in ("replicated", "sharded"):
        raise ConfigError(f"data must be 'replicated' or 'sharded', got {data!r}")
    sharded = data == "sharded" and world > 1
    n = buffer["obs"].shape[0]
    adv = buffer["advantages"].to(torch.float32)
    if config.normalize_advantages:
        if sharded:  # global mean / std over every rank's buffer (one tiny all-reduce)
            a64 = buffer["advantages"].to(torch.float64)
            mom = torch.stack([a64.sum(), (a64 * a64).sum(), torch.tensor(float(n), dtype=torch.float64,
                                                                           device=a64.device)])
            dist.all_reduce(mom, op=dist.ReduceOp.SUM, group=reducer.group if reducer is not None else None)
            N = mom[2]
            mean = mom[0] / N
            std = torch.sqrt(torch.clamp(mom[1] / N - mean * mean, min=0.0))  # population std
            adv = ((buffer["advantages"].to(torch.float64) - mean) / (std + 1e-8)).to(torch.float32)
        else:
            # numpy's std (ddof=0) on the float32 advantages, as trainer.py:171-173 computes it
            adv = (adv - adv.mean()) / (adv.std(correction=0) + 1e-8)
    flat = {"obs": buffer["obs"], "actions": buffer["actions"], "old_log_probs": buffer["log_probs"],
            "advantages": adv, "returns": buffer["returns"].to(torch.float32)}
    if bundle.mode == "ac_mpc":
        flat["x_init"] = buffer["x_init"]
        flat["U_warm"] = buffer["U_warm"]
    if sharded:
        mb = max(1, min(config.minibatch_size, n * world) // world)
    else:
        mb = min(config.minibatch_size, n)
    stats_sink, skipped, last = {}, 0, {}
    for _ in range(config.sgd_epochs):
        perm = torch.randperm(n, generator=generator).to(buffer["obs"].device)
        for start in range(0, n, mb):
            sel = perm[start:start + mb]
            if not sharded:
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
    last["samples_trained"] = n * config.sgd_epochs * (world if sharded else 1)
    return last
