"""Loading the committed golden fixtures (tests/golden/*.npz, produced from the
unmodified reference by tests/golden/make_golden.py)."""

from __future__ import annotations

import glob
import os
from dataclasses import dataclass

import numpy as np

from paper_2605_29155_b200 import _abi
from paper_2605_29155_b200.dynamics import DynModel
from paper_2605_29155_b200.settings import SolveSettings

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
SOLVE_CASES = sorted(
    os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN_DIR, "*.npz"))
    if os.path.basename(p) not in ("boxqp.npz", "dynamics.npz", "raceenv.npz", "ppo.npz")
)


@dataclass
class Golden:
    name: str
    model: DynModel
    settings: SolveSettings
    layout: str
    d: dict

    def __getitem__(self, k):
        return self.d[k]

    @property
    def B(self):
        return self.d["x0"].shape[0]

    def C_dense(self):
        if "C" in self.d:
            return self.d["C"]
        diag = self.d["diag"]
        B, T, nz = diag.shape
        C = np.zeros((B, T, nz, nz))
        idx = np.arange(nz)
        C[:, :, idx, idx] = diag
        return C

    def cost(self, layout: int):
        """Cost tensor in the requested ABI layout (diag only for diagonal problems)."""
        if layout == _abi.COST_DIAG:
            return self.d["diag"]
        return self.C_dense()

    def layouts(self):
        return [_abi.COST_DENSE, _abi.COST_DIAG] if "diag" in self.d else [_abi.COST_DENSE]

    def dC_in(self, layout: int):
        dC = self.d["dC"]
        if layout == _abi.COST_DIAG:
            idx = np.arange(dC.shape[-1])
            return dC[:, :, idx, idx]
        return dC


def load(name: str) -> Golden:
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    d = {k: z[k] for k in z.files}
    model = DynModel(kind=int(d["kind"]), dt=float(d["dt"]), n_x=int(d["nx"]), n_u=int(d["nu"]),
                     params=d["params"])
    settings = SolveSettings(T=int(d["T"]), u_min=d["u_min"], u_max=d["u_max"],
                             K_max=int(d["K_max"]), alphas=tuple(d["alphas"]),
                             conv_tol=float(d["conv_tol"]),
                             boxqp_max_iter=int(d["boxqp_max_iter"]),
                             boxqp_tol=float(d["boxqp_tol"]))
    return Golden(name, model, settings, str(d["layout"]), d)


def load_aux(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN_DIR, f"{name}.npz"))
    return {k: z[k] for k in z.files}
