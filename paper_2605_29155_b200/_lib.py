"""Loader for libdiffmpc.so (the in-tree CUDA library behind include/diffmpc.h).

Fails loudly: if the shared object is missing, or no CUDA device is present when a
compute entry point is used, an ExtensionMissingError is raised. There is no CPU
fallback anywhere in the product path.
"""

from __future__ import annotations

import ctypes
import os
import threading

from . import _abi
from .errors import ConfigError, ExtensionMissingError

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libdiffmpc.so")
# development A/B aid: load another in-tree build of the same ABI (tools/ab_*.sh)
if os.environ.get("DIFFMPC_LIB"):
    LIB_PATH = os.path.abspath(os.environ["DIFFMPC_LIB"])
_lock = threading.Lock()
_lib = None

EXPORTS = (
    "diffmpc_forward_f32", "diffmpc_forward_f64", "diffmpc_backward_f32", "diffmpc_backward_f64",
    "diffmpc_dynamics_f32", "diffmpc_dynamics_f64", "diffmpc_supported", "diffmpc_launch_count",
    "diffmpc_last_error", "diffmpc_abi_version", "diffmpc_race_step_f64",
)


def lib():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ExtensionMissingError(
                f"{LIB_PATH} is not built; run `python -m paper_2605_29155_b200.build` "
                "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp = ctypes.c_void_p
        for dt in ("f32", "f64"):
            f = getattr(L, f"diffmpc_forward_{dt}")
            f.argtypes = [vp, vp, vp]
            f.restype = ctypes.c_int
            f = getattr(L, f"diffmpc_backward_{dt}")
            f.argtypes = [vp, vp, vp]
            f.restype = ctypes.c_int
            f = getattr(L, f"diffmpc_dynamics_{dt}")
            f.argtypes = [vp, ctypes.c_int32, vp, vp, vp, vp, vp, vp, vp]
            f.restype = ctypes.c_int
        L.diffmpc_race_step_f64.argtypes = [vp, ctypes.c_int32, ctypes.c_int32, ctypes.c_double] + [vp] * 11
        L.diffmpc_race_step_f64.restype = ctypes.c_int
        L.diffmpc_forward_workspace_bytes.argtypes = [vp, ctypes.c_int32]
        L.diffmpc_forward_workspace_bytes.restype = ctypes.c_uint64
        L.diffmpc_supported.argtypes = [ctypes.c_int32] * 3
        L.diffmpc_supported.restype = ctypes.c_int
        L.diffmpc_launch_count.argtypes = []
        L.diffmpc_launch_count.restype = ctypes.c_int64
        L.diffmpc_last_error.argtypes = []
        L.diffmpc_last_error.restype = ctypes.c_char_p
        L.diffmpc_abi_version.argtypes = []
        L.diffmpc_abi_version.restype = ctypes.c_int32
        if L.diffmpc_abi_version() != _abi.ABI_VERSION:
            raise ExtensionMissingError("libdiffmpc.so ABI version mismatch; rebuild it")
        _lib = L
        return _lib


def check(rc: int):
    if rc != 0:
        msg = lib().diffmpc_last_error().decode()
        raise ConfigError(msg)


_replayed = 0  # DiffMPC kernels executed by CUDA-graph replays (invisible to the C counter)


def note_graph_replay(n: int):
    """Account the n DiffMPC launches a captured graph performs per replay."""
    global _replayed
    _replayed += int(n)


def launch_count() -> int:
    """DiffMPC kernels launched so far: ABI calls (captures included) + graph replays."""
    return int(lib().diffmpc_launch_count()) + _replayed


def supported(kind: int, nx: int, nu: int) -> bool:
    return bool(lib().diffmpc_supported(kind, nx, nu))
