"""Shared parity comparison (GPU kernels vs the oracle / the reference goldens).

Used by the -m gpu parity tests and by tools/parity_report.py (which writes the measured
per-case errors to profiles/). The gate is SURVEY.md §8(c) / BASELINE.json north_star:
per instance and tensor  max|a-b| <= tol * max(1, max|b|)  (tol 1e-4 for the f32 kernels,
1e-9 for f64), identical clamp masks, iteration counts, convergence / failure flags and
step-size histories.
"""

from __future__ import annotations

import numpy as np
import torch

TOL = {torch.float64: 1e-9, torch.float32: 1e-4}

FWD_KEYS = ("X", "U", "J", "K", "k", "J_hist")
BWD_KEYS = ("dC", "dc", "dx0", "dX", "dU")


def rel_err(a, b):
    """Per-instance max|a-b| / max(1, max|b|) over the trailing dims."""
    a = np.asarray(a, dtype=np.float64).reshape(a.shape[0], -1)
    b = np.asarray(b, dtype=np.float64).reshape(b.shape[0], -1)
    if a.shape[1] == 0 or a.shape[0] == 0:
        return np.zeros(a.shape[0])
    return np.abs(a - b).max(1) / np.maximum(1.0, np.abs(b).max(1))


def as_np(t):
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        t = t.detach().cpu()
        if t.dtype == torch.bool:
            t = t.to(torch.uint8)
        return t.numpy()
    return np.asarray(t)


def round_inputs(arrs, dtype):
    """The inputs exactly as the kernel of `dtype` sees them (f32 kernels: rounded to f32),
    so GPU and oracle solve IDENTICAL problems."""
    if dtype == torch.float64:
        return [None if a is None else np.asarray(a, np.float64) for a in arrs]
    return [None if a is None else np.asarray(a, np.float32).astype(np.float64) for a in arrs]


def decision_margin(ref, i, conv_tol):
    """Oracle-side margin of the convergence decision of instance i at its last iteration:
    (rel - conv_tol) / conv_tol, where rel = |J_prev - J| / max(1, |J_prev|)
    (ilqr.py:233-238). Small |margin| = the reference decided within round-off."""
    it = int(ref["iters"][i])
    if it == 0:
        return float("nan")
    Jh = ref["J_hist"][i]
    jp, jn = Jh[it - 1], Jh[it]
    rel = abs(jp - jn) / max(1.0, abs(jp))
    return (rel - conv_tol) / conv_tol if conv_tol > 0 else float("nan")


def compare_forward(out, ref, dtype, conv_tol=1e-6, check_gains=True):
    """Compare a SolveOutput with an oracle / golden dict. Returns a report dict:
    flips (instances whose iteration count differs), worst per-tensor errors over the
    instances with identical counts, and mismatch counts of the discrete outputs."""
    it = as_np(out.iters)
    flips = np.nonzero(it != ref["iters"])[0]
    fail_ref = ref["fail_t"] >= 0
    ok = ~fail_ref & (ref["diverged"] == 0)
    same = ok & (it == ref["iters"])
    rep = {"B": int(it.shape[0]), "flips": flips.tolist(),
           "flip_margins": [decision_margin(ref, int(i), conv_tol) for i in flips[:32]],
           "fail_mismatch": int(((as_np(out.fail_t) >= 0) != fail_ref).sum()),
           "fail_t_mismatch": int((as_np(out.fail_t)[fail_ref] != ref["fail_t"][fail_ref]).sum()),
           "diverged_mismatch": int((as_np(out.diverged).astype(np.uint8) != ref["diverged"]).sum()),
           "n_compared": int(same.sum())}
    err = {}
    for key in FWD_KEYS:
        if key in ("K", "k") and (not check_gains or getattr(out, key, None) is None):
            continue
        a = as_np(getattr(out, key))
        b = np.asarray(ref[key])
        if key == "J":
            a, b = a[:, None], b[:, None]
        e = rel_err(a[same], b[same])
        err[key] = float(e.max(initial=0.0))
    rep["err"] = err
    rep["clamp_mismatch"] = int((as_np(out.clamped).astype(np.uint8)[same] != ref["clamped"][same]).any(
        axis=tuple(range(1, ref["clamped"].ndim))).sum())
    rep["converged_mismatch"] = int((as_np(out.converged).astype(np.uint8)[same] != ref["converged"][same]).sum())
    # the accepted step sizes are discrete: equal after rounding to the kernel's type
    ah = as_np(out.alpha_hist).astype(np.float64)
    rh = np.asarray(ref["alpha_hist"], np.float64)
    if dtype == torch.float32:
        rh = rh.astype(np.float32).astype(np.float64)
    rep["alpha_hist_mismatch"] = int((ah[same] != rh[same]).any(axis=1).sum())
    return rep


def compare_backward(g, ref, dtype, mask, layout_diag=False):
    """Compare a GradOutput (want_traj=True) with an oracle / golden gradient dict on the
    instances in `mask` (typically: identical forward counts, not failed)."""
    bf_ref = np.asarray(ref["bfail_t"] if "bfail_t" in ref else ref["fail_t"])  # golden | oracle dict
    rep = {"bfail_mismatch": int((as_np(g.fail_t) != bf_ref).sum())}
    ok = mask & (bf_ref < 0)
    err = {}
    for key in BWD_KEYS:
        a = as_np(getattr(g, key))
        if a is None:
            continue
        b = np.asarray(ref[key])
        if key == "dC" and layout_diag and b.ndim == 4:
            idx = np.arange(b.shape[-1])
            b = b[:, :, idx, idx]
        err[key] = float(rel_err(a[ok], b[ok]).max(initial=0.0))
    rep["err"] = err
    bfail = bf_ref >= 0
    rep["failed_nonzero"] = int(sum(np.any(as_np(getattr(g, k))[bfail] != 0.0) for k in ("dC", "dc", "dx0")))
    rep["n_compared"] = int(ok.sum())
    return rep


def assert_forward(rep, dtype, allow_flips=False, xtol=None):
    tol = TOL[dtype] if xtol is None else xtol
    assert rep["fail_mismatch"] == 0 and rep["fail_t_mismatch"] == 0, rep
    assert rep["diverged_mismatch"] == 0, rep
    if not allow_flips:
        assert not rep["flips"], f"iteration counts differ at {rep['flips'][:16]} (margins {rep['flip_margins'][:8]})"
    for key, e in rep["err"].items():
        assert e <= tol, f"{key}: worst rel err {e:.3e} > {tol:g}"
    assert rep["clamp_mismatch"] == 0, f"clamp masks differ on {rep['clamp_mismatch']} instances"
    assert rep["alpha_hist_mismatch"] == 0, f"step-size histories differ on {rep['alpha_hist_mismatch']} instances"


def assert_backward(rep, dtype, tol=None):
    tol = TOL[dtype] if tol is None else tol
    assert rep["bfail_mismatch"] == 0, rep
    assert rep["failed_nonzero"] == 0, "failed instances must get zero gradients"
    for key, e in rep["err"].items():
        assert e <= tol, f"{key}: worst rel err {e:.3e} > {tol:g}"
