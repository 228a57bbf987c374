"""ctypes binding of liblloydkit_b200.so (the C ABI in include/lloydkit_b200.h).

There is no fallback: if the library is missing or no CUDA device is present,
every entry point raises.  The library has no torch types in its signatures;
torch only provides the device workspace, the stream handle and (multi-GPU)
the NCCL all-reduce of the int64 delta buffer.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblloydkit_b200.so")
CSRC = os.path.join(_HERE, "csrc")

LK_OK, LK_ERR_ARG, LK_ERR_CUDA, LK_ERR_STATE, LK_ERR_UNSUPPORTED = 0, 1, 2, 3, 4

STRAT_IDS = {"lloyd": 0, "hamerly": 1, "yinyang": 2, "elkan": 3, "regroup": 4}
KERNEL_IDS = {"auto": 0, "simt": 1, "tc": 2}

BUF = {"x32": 0, "x64": 1, "c64": 2, "labels": 3, "ub": 4, "lb": 5, "delta": 6, "stats": 7,
       "sse": 8, "group_of": 9, "counts": 10, "qexp": 11, "hlog": 12, "hlog_off": 13,
       "tstamp": 14}
NSTAT = 16
STAT = {"changed": 0, "flagged": 1, "active": 2, "work": 3, "dist": 4, "bound_upd": 5,
        "candidate": 6, "changed_global": 7, "overflow": 8, "ywl": 9, "pairs": 10,
        "regrouped": 11}

# Every symbol the header declares (checked by tests/test_native_abi.py).
EXPORTED = (
    "lk_version", "lk_last_error", "lk_workspace_bytes", "lk_ctx_create", "lk_ctx_destroy",
    "lk_buffer", "lk_layout", "lk_scan_points", "lk_set_quant", "lk_set_centroids",
    "lk_set_groups", "lk_step_assign", "lk_step_update", "lk_graph_capture", "lk_graph_replay",
    "lk_launch_count", "lk_profile", "lk_profile_read", "lk_d2_update", "lk_group_shape",
    "lk_validate_bounds",
)


class LkConfig(ctypes.Structure):
    _fields_ = [
        ("n_local", ctypes.c_int64),
        ("n_total", ctypes.c_int64),
        ("d", ctypes.c_int32),
        ("k", ctypes.c_int32),
        ("strategy", ctypes.c_int32),
        ("groups", ctypes.c_int32),
        ("t_max", ctypes.c_int32),
        ("kernel", ctypes.c_int32),
        ("has_x64", ctypes.c_int32),
        ("device", ctypes.c_int32),
        ("history_cap", ctypes.c_int64),
        ("ranks", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class NativeError(RuntimeError):
    pass


_lib = None


def build(verbose: bool = False) -> str:
    """Compile the CUDA sources for sm_100a (nvcc cross-compiles without a GPU)."""
    r = subprocess.run(["make", "-C", CSRC, "-j8"], capture_output=not verbose, text=True)
    if r.returncode != 0:
        raise NativeError("building liblloydkit_b200.so failed:\n" + (r.stdout or "")
                          + (r.stderr or ""))
    return LIB_PATH


def load():
    """Load the shared library (no GPU needed to load it)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise NativeError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                          "(or make -C paper_2010_06654_b200/csrc)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64
    cfgp = ctypes.POINTER(LkConfig)
    L.lk_version.restype = i32
    L.lk_last_error.restype = ctypes.c_char_p
    L.lk_workspace_bytes.argtypes = [cfgp, ctypes.POINTER(u64)]
    L.lk_ctx_create.argtypes = [ctypes.POINTER(vp), cfgp, vp, u64]
    L.lk_ctx_destroy.argtypes = [vp]
    L.lk_buffer.argtypes = [vp, i32, ctypes.POINTER(u64), ctypes.POINTER(u64)]
    L.lk_layout.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i32)]
    L.lk_group_shape.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32)]
    L.lk_validate_bounds.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double), i32, vp]
    L.lk_scan_points.argtypes = [vp, vp]
    L.lk_set_quant.argtypes = [vp, vp]
    L.lk_set_centroids.argtypes = [vp, vp, vp]
    L.lk_set_groups.argtypes = [vp, vp, vp]
    L.lk_step_assign.argtypes = [vp, i32, vp]
    L.lk_step_update.argtypes = [vp, i32, vp]
    L.lk_graph_capture.argtypes = [vp, i32, vp]
    L.lk_graph_replay.argtypes = [vp, vp]
    L.lk_launch_count.argtypes = [vp]
    L.lk_launch_count.restype = i64
    L.lk_profile.argtypes = [vp, i32]
    L.lk_profile_read.argtypes = [vp, i32, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(i64)]
    L.lk_d2_update.argtypes = [vp, vp, i64, i32, i64, vp, vp, i32, vp]
    for name in ("lk_workspace_bytes", "lk_ctx_create", "lk_ctx_destroy", "lk_buffer",
                 "lk_layout", "lk_scan_points", "lk_set_quant", "lk_set_centroids",
                 "lk_set_groups", "lk_step_assign", "lk_step_update", "lk_graph_capture",
                 "lk_graph_replay", "lk_profile", "lk_profile_read", "lk_d2_update",
                 "lk_group_shape", "lk_validate_bounds"):
        getattr(L, name).restype = i32
    _lib = L
    return L


def check(status: int, what: str):
    if status != LK_OK:
        msg = load().lk_last_error().decode(errors="replace")
        if status == LK_ERR_ARG:
            from .core import ContractError
            raise ContractError(f"{what}: {msg}")
        raise NativeError(f"{what} failed (status {status}): {msg}")
