"""Per-entry FD vs analytic gradients of the MPC module on linear dynamics (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2605_29155_b200.mpc import MPC, QuadCost, LinDx
rng = np.random.default_rng(2)
n, m, T, B = 3, 2, 5, 2
A = torch.tensor(np.eye(n) + 0.1 * rng.normal(size=(n, n)), device="cuda")
Bm = torch.tensor(0.5 * rng.normal(size=(n, m)), device="cuda")
M = rng.normal(size=(T, B, n + m, n + m))
C = torch.tensor(0.3 * np.einsum("tbij,tbkj->tbik", M, M) + 0.8 * np.eye(n + m), device="cuda", requires_grad=True)
c = torch.tensor(0.3 * rng.normal(size=(T, B, n + m)), device="cuda", requires_grad=True)
x0 = torch.tensor(0.5 * rng.normal(size=(B, n)), device="cuda", requires_grad=True)
dx = LinDx(A, Bm, learn=True).cuda()
mpc = MPC(n, m, T, u_lower=-0.25, u_upper=0.25, lqr_iter=60, eps=1e-14)
torch.manual_seed(0)
wx, wu = torch.randn(T, B, n, device="cuda", dtype=torch.float64), torch.randn(T, B, m, device="cuda", dtype=torch.float64)
for wJ, wxs, wus in ((0.3, 1, 1), (0.0, 1, 0), (0.0, 0, 1), (1.0, 0, 0)):
    for tt in (C, c, x0, dx.params):
        tt.grad = None
    def loss():
        x, u, J = mpc(x0, QuadCost(C, c), dx)
        return wxs * (wx * x).sum() + wus * (wu * u).sum() + wJ * J.sum()
    loss().backward()
    print("weights J,x,u", wJ, wxs, wus)
    for name, t, idx in [("C", C, (1, 0, 2, 2)), ("C", C, (3, 1, 0, 4)), ("c", c, (0, 1, 3)), ("c", c, (4, 0, 1)), ("x0", x0, (1, 2)),
                         ("th", dx.params, (0,)), ("th", dx.params, (10,))]:
        idxs = [idx]
        if t is C and idx[2] != idx[3]:
            idxs.append((idx[0], idx[1], idx[3], idx[2]))
        eps = 1e-6
        with torch.no_grad():
            for i in idxs: t[i] += eps
            up = float(loss())
            for i in idxs: t[i] -= 2 * eps
            dn = float(loss())
            for i in idxs: t[i] += eps
        fd = (up - dn) / (2 * eps)
        an = sum(float(t.grad[i]) for i in idxs)
        print(f"  {name}{idx}: fd {fd:+.8e} an {an:+.8e} rel {abs(fd-an)/max(1e-3,abs(fd)):.2e}")
x, u, J = mpc(x0, QuadCost(C, c), dx)
print("u", u[:, :, :].detach().cpu().numpy().round(4).tolist())
