"""The C-ABI library loads, exports every entry point include/diffmpc.h declares, its struct
layout matches the header, and configuration errors are rejected before any device work
(so these run without a GPU)."""

import ctypes
import os
import re
import subprocess
import tempfile

import numpy as np
import pytest

from paper_2605_29155_b200 import _abi, _lib
from paper_2605_29155_b200.dynamics import DynModel
from paper_2605_29155_b200.settings import SolveSettings

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "diffmpc.h")


def declared_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|int32_t|uint64_t|const char\*)\s+(diffmpc_\w+)\s*\(", txt, re.M)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    names = declared_functions()
    assert len(names) >= 10
    for n in names:
        assert hasattr(L, n), f"{n} declared in diffmpc.h but not exported"
    nm = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", nm), n


def test_abi_version_and_supported_table():
    assert _lib.lib().diffmpc_abi_version() == _abi.ABI_VERSION
    assert _lib.supported(3, 13, 4)
    assert _lib.supported(1, 6, 2)
    assert _lib.supported(2, 3, 2)
    assert not _lib.supported(3, 12, 4)


def test_struct_layout_matches_header():
    src = r'''
#include <stdio.h>
#include <stddef.h>
#include "diffmpc.h"
int main(void) {
  printf("%zu %zu %zu %zu %zu %zu %zu %zu %zu %zu %zu\n", sizeof(DiffMPCProblem), offsetof(DiffMPCProblem, dt),
         offsetof(DiffMPCProblem, u_min), offsetof(DiffMPCProblem, alphas), sizeof(DiffMPCForwardIO),
         sizeof(DiffMPCBackwardIO), offsetof(DiffMPCBackwardIO, fail_t), sizeof(DiffMPCTrack),
         offsetof(DiffMPCTrack, width), offsetof(DiffMPCTrack, k_p), offsetof(DiffMPCTrack, omega_scale));
  return 0;
}
'''
    d = tempfile.mkdtemp()
    c = os.path.join(d, "l.c")
    open(c, "w").write(src)
    exe = os.path.join(d, "l")
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe], check=True)
    got = [int(v) for v in subprocess.run([exe], capture_output=True, text=True).stdout.split()]
    P, F, Bk, Tr = _abi.DiffMPCProblem, _abi.DiffMPCForwardIO, _abi.DiffMPCBackwardIO, _abi.DiffMPCTrack
    want = [ctypes.sizeof(P), P.dt.offset, P.u_min.offset, P.alphas.offset, ctypes.sizeof(F),
            ctypes.sizeof(Bk), Bk.fail_t.offset, ctypes.sizeof(Tr), Tr.width.offset, Tr.k_p.offset,
            Tr.omega_scale.offset]
    assert got == want


def _problem(**kw):
    m = DynModel.quadrotor()
    s = SolveSettings(T=10, u_min=np.zeros(4), u_max=np.full(4, 5.0))
    p = _abi.make_problem(m, s, 4, _abi.COST_DENSE)
    for k, v in kw.items():
        setattr(p, k, v)
    return p


@pytest.mark.parametrize("field,value,msg", [
    ("T", 0, "horizon"), ("K_max", 0, "K_max"), ("n_alpha", 0, "n_alpha"), ("nu", 9, "n_u"),
    ("cost_layout", 7, "layout"), ("dt", -1.0, "dt"),
])
def test_config_errors_rejected_without_device_work(field, value, msg):
    L = _lib.lib()
    p = _problem(**{field: value})
    io = _abi.DiffMPCForwardIO()
    rc = L.diffmpc_forward_f32(ctypes.byref(p), ctypes.byref(io), None)
    assert rc < 0
    assert msg in L.diffmpc_last_error().decode()


def test_bad_bounds_and_alphas_rejected():
    L = _lib.lib()
    p = _problem()
    p.u_min[0], p.u_max[0] = 1.0, 0.0
    assert L.diffmpc_forward_f64(ctypes.byref(p), ctypes.byref(_abi.DiffMPCForwardIO()), None) < 0
    p = _problem()
    p.alphas[1] = 2.0
    assert L.diffmpc_backward_f32(ctypes.byref(p), ctypes.byref(_abi.DiffMPCBackwardIO()), None) < 0
    assert "alphas" in L.diffmpc_last_error().decode()


def test_unsupported_shape_rejected():
    L = _lib.lib()
    p = _problem(nx=12)
    rc = L.diffmpc_forward_f32(ctypes.byref(p), ctypes.byref(_abi.DiffMPCForwardIO()), None)
    assert rc < 0 and "no compiled kernels" in L.diffmpc_last_error().decode()


def test_wrong_parameter_count_rejected():
    L = _lib.lib()
    p = _problem(n_theta=3)
    rc = L.diffmpc_forward_f32(ctypes.byref(p), ctypes.byref(_abi.DiffMPCForwardIO()), None)
    assert rc < 0 and "parameters" in L.diffmpc_last_error().decode()


def test_null_required_pointer_rejected():
    L = _lib.lib()
    p = _problem()
    rc = L.diffmpc_forward_f32(ctypes.byref(p), ctypes.byref(_abi.DiffMPCForwardIO()), None)
    assert rc < 0 and "NULL" in L.diffmpc_last_error().decode()


def test_forward_workspace_bytes_matches_layout():
    """diffmpc_forward_workspace_bytes: 256-byte counter block + per-problem 128-byte aligned
    gain rows (T x n_u x LDA) and stage records ([C_t padded | c_t padded])."""
    import ctypes

    from paper_2605_29155_b200 import DynModel, SolveSettings

    L = _lib.lib()
    m = DynModel.quadrotor()
    st = SolveSettings(T=10, u_min=0.0, u_max=5.886)
    rup = lambda v, a: (v + a - 1) // a * a  # noqa: E731
    for layout, B in ((_abi.COST_DENSE, 3), (_abi.COST_DIAG, 5)):
        p = _abi.make_problem(m, st, B, layout)
        for elem in (4, 8):
            vn = 16 // elem
            lda, zld = rup(13, vn), rup(17, vn)
            rec = (zld if layout == _abi.COST_DIAG else 17 * zld) + zld
            want = 256 + B * (rup(10 * 4 * lda * elem, 128) + rup(10 * rec * elem, 128))
            assert L.diffmpc_forward_workspace_bytes(ctypes.byref(p), elem) == want
    assert L.diffmpc_forward_workspace_bytes(ctypes.byref(p), 3) == 0
