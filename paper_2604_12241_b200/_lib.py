"""ctypes binding of libtempmine_b200.so (include/tempmine_b200.h).

The library is the only compute path: if it is missing or fails to load,
every entry point raises — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libtempmine_b200.so"

# enum tm_family
TM_FAN, TM_DEGREE, TM_CYCLE, TM_SG, TM_GS, TM_STACK = 1, 2, 3, 4, 5, 6
FAMILY_NAMES = {TM_FAN: "FAN", TM_DEGREE: "DEGREE", TM_CYCLE: "CYCLE", TM_SG: "SG",
                TM_GS: "GS", TM_STACK: "STACK"}

# enum tm_status
TM_OK = 0
TM_E_CUDA, TM_E_OOM, TM_E_BAD_ARG, TM_E_UNSUPPORTED_PLAN, TM_E_OVERFLOW, TM_E_STATE = -1, -2, -3, -4, -5, -6
MAX_PLANS = 32


class TmPlanDesc(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("endpoint", ctypes.c_int32),
                ("direction", ctypes.c_int32), ("exclude_trigger", ctypes.c_int32),
                ("cycle_len", ctypes.c_int32), ("min_size", ctypes.c_int32),
                ("delta", ctypes.c_int64)]


class TmGraphInfo(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("n_edges", ctypes.c_int64),
                ("n_ranks", ctypes.c_int64), ("max_out_degree", ctypes.c_int64),
                ("max_in_degree", ctypes.c_int64), ("n_selfloops", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("device", ctypes.c_int32),
                ("rank_bits", ctypes.c_int32), ("node_bits", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class TmMineStats(ctypes.Structure):
    _fields_ = [("triggers", ctypes.c_int64), ("heavy_triggers", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("light_ms", ctypes.c_float),
                ("heavy_ms", ctypes.c_float), ("total_ms", ctypes.c_float),
                ("reserved", ctypes.c_int32)]


# name -> (restype, argtypes): every symbol include/tempmine_b200.h declares
_P = ctypes.c_void_p
_I64P = ctypes.POINTER(ctypes.c_int64)
SIGNATURES = {
    "tm_abi_version": (ctypes.c_int, []),
    "tm_graph_build": (ctypes.c_int, [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, _P, _P, _P,
                                      ctypes.c_int, _P, ctypes.POINTER(_P)]),
    "tm_graph_info_get": (ctypes.c_int, [_P, ctypes.POINTER(TmGraphInfo)]),
    "tm_graph_export_csr": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P, _P]),
    "tm_graph_degrees": (ctypes.c_int, [_P, ctypes.c_int, _P]),
    "tm_mine": (ctypes.c_int, [_P, ctypes.POINTER(TmPlanDesc), ctypes.c_int, ctypes.c_int64,
                               ctypes.c_int64, _P, ctypes.c_int, _P]),
    "tm_mine_members": (ctypes.c_int, [_P, ctypes.POINTER(TmPlanDesc), ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, _P, ctypes.c_int, _P]),
    "tm_last_mine_stats": (ctypes.c_int, [_P, ctypes.POINTER(TmMineStats)]),
    "tm_csv_format": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(ctypes.c_int64)]),
    "tm_csv_fetch": (ctypes.c_int, [_P, _P, ctypes.c_int64]),
    "tm_set_profiling": (ctypes.c_int, [_P, ctypes.c_int]),
    "tm_kernel_launch_count": (ctypes.c_int64, []),
    "tm_last_error": (ctypes.c_char_p, []),
    "tm_graph_free": (None, [_P]),
}
ABI_VERSION = 2


class TempmineError(RuntimeError):
    """A C-ABI call failed; `code` is the tm_status value."""

    def __init__(self, code: int, message: str):
        self.code = code
        super().__init__(f"[tm status {code}] {message}")


class UnsupportedPlanError(TempmineError):
    """TM_E_UNSUPPORTED_PLAN — the plan is not one of the GPU families."""


_lock = threading.Lock()
_lib: ctypes.CDLL | None = None


def load(path: str | os.PathLike | None = None) -> ctypes.CDLL:
    """Load the shared library once; raises if it is absent (no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        p = Path(path) if path else Path(os.environ.get("TM_LIB", LIB_PATH))
        if not p.exists():
            raise RuntimeError(
                f"{p} is missing: build it with `python -m paper_2604_12241_b200.build` "
                "(nvcc, sm_100a). The mining path has no CPU fallback.")
        lib = ctypes.CDLL(str(p))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        if lib.tm_abi_version() != ABI_VERSION:
            raise RuntimeError(f"ABI mismatch: library {lib.tm_abi_version()} vs wrapper {ABI_VERSION}")
        _lib = lib
        return lib


def check(rc: int, what: str) -> None:
    if rc == TM_OK:
        return
    msg = load().tm_last_error().decode("utf-8", "replace")
    cls = UnsupportedPlanError if rc == TM_E_UNSUPPORTED_PLAN else TempmineError
    if rc == TM_E_BAD_ARG:
        raise ValueError(f"{what}: {msg}")
    raise cls(rc, f"{what}: {msg}")


def ptr(a: np.ndarray | None) -> int | None:
    if a is None:
        return None
    return a.ctypes.data


def plan_array(descs) -> ctypes.Array:
    arr = (TmPlanDesc * max(len(descs), 1))()
    for i, d in enumerate(descs):
        arr[i] = TmPlanDesc(d.family, d.endpoint, d.direction, d.exclude_trigger,
                            d.cycle_len, d.min_size, d.delta)
    return arr


def kernel_launch_count() -> int:
    return int(load().tm_kernel_launch_count())
