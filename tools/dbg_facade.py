import sys; sys.path[:0]=['.','oracle','tests']
import numpy as np, torch
from paper_2605_29155_b200.mpc import MPC, LinDx, QuadCost
rng = np.random.default_rng(2)
n, m, T, B = 3, 2, 5, 2
A = torch.tensor(np.eye(n) + 0.1 * rng.normal(size=(n, n)), device="cuda")
Bm = torch.tensor(0.5 * rng.normal(size=(n, m)), device="cuda")
M = rng.normal(size=(T, B, n + m, n + m))
C = torch.tensor(0.3 * np.einsum("tbij,tbkj->tbik", M, M) + 0.8 * np.eye(n + m), device="cuda", requires_grad=True)
c = torch.tensor(0.3 * rng.normal(size=(T, B, n + m)), device="cuda", requires_grad=True)
x0 = torch.tensor(0.5 * rng.normal(size=(B, n)), device="cuda", requires_grad=True)
dx = LinDx(A, Bm, learn=True).cuda()
for ub in (0.25, 1e3):
  for terms in ("x", "u", "J"):
    mpc = MPC(n, m, T, u_lower=-ub, u_upper=ub, lqr_iter=60, eps=1e-14)
    g = torch.Generator("cuda").manual_seed(1)
    wx, wu = torch.randn(T, B, n, device="cuda", dtype=torch.float64, generator=g), torch.randn(T, B, m, device="cuda", dtype=torch.float64, generator=g)
    def loss():
        x, u, J = mpc(x0, QuadCost(C, c), dx)
        return {"x": (wx * x).sum(), "u": (wu * u).sum(), "J": 0.3 * J.sum()}[terms]
    for t in (C, c, x0, dx.params):
        t.grad = None
    loss().backward()
    eps = 1e-6
    out = []
    for name, t, idx in [("C", C, (1, 0, 2, 2)), ("C", C, (3, 1, 0, 4)), ("c", c, (0, 1, 3)), ("c", c, (4, 0, 1)), ("x0", x0, (1, 2)), ("th", dx.params, (0,)), ("th", dx.params, (10,))]:
        with torch.no_grad():
            t[idx] += eps; up = float(loss()); t[idx] -= 2 * eps; dn = float(loss()); t[idx] += eps
        fd = (up - dn) / (2 * eps); an = float(t.grad[idx])
        out.append(f"{name}{idx}: fd {fd:+.6f} an {an:+.6f}")
    print("bound", ub, "loss", terms, "clamped", int(mpc.last_result.clamped.sum()), " | ".join(out))
