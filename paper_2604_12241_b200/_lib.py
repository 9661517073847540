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


VM_MAX_CELLS, VM_MAX_OPS, VM_MAX_PREDS, VM_MAX_SYMS, VM_TABLE = 8, 4, 8, 16, 1024


class TmVmPred(ctypes.Structure):
    _fields_ = [("cmp", ctypes.c_int32), ("lk", ctypes.c_int32), ("lref", ctypes.c_int32),
                ("rk", ctypes.c_int32), ("rref", ctypes.c_int32), ("table", ctypes.c_int32),
                ("sym", ctypes.c_int32), ("pad", ctypes.c_int32), ("lnum", ctypes.c_double),
                ("rnum", ctypes.c_double)]


class TmVmOperand(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("var", ctypes.c_int32), ("slot", ctypes.c_int32),
                ("dir", ctypes.c_int32), ("sym", ctypes.c_int32)]


class TmVmCell(ctypes.Structure):
    _fields_ = [("op", ctypes.c_int32), ("parent", ctypes.c_int32), ("forward", ctypes.c_int32),
                ("n_ops", ctypes.c_int32), ("ops", TmVmOperand * VM_MAX_OPS),
                ("n_node", ctypes.c_int32), ("n_edge", ctypes.c_int32), ("n_gate", ctypes.c_int32),
                ("n_order", ctypes.c_int32), ("node", (ctypes.c_int32 * 3) * VM_MAX_PREDS),
                ("edge", TmVmPred * VM_MAX_PREDS), ("gate", TmVmPred * VM_MAX_PREDS),
                ("order", (ctypes.c_int32 * 3) * VM_MAX_PREDS)]


class TmVmProgram(ctypes.Structure):
    _fields_ = [("n_cells", ctypes.c_int32), ("mode", ctypes.c_int32), ("min_size", ctypes.c_int32),
                ("target", ctypes.c_int32 * 2), ("uses_attrs", ctypes.c_int32), ("delta", ctypes.c_int64),
                ("cells", TmVmCell * VM_MAX_CELLS), ("table", ctypes.c_int8 * VM_TABLE)]


class TmGraphInfo(ctypes.Structure):
    _fields_ = [("n_nodes", ctypes.c_int64), ("n_edges", ctypes.c_int64),
                ("n_ranks", ctypes.c_int64), ("max_out_degree", ctypes.c_int64),
                ("max_in_degree", ctypes.c_int64), ("n_selfloops", ctypes.c_int64),
                ("device_bytes", ctypes.c_int64), ("device", ctypes.c_int32),
                ("rank_bits", ctypes.c_int32), ("node_bits", ctypes.c_int32),
                ("prep_ms", ctypes.c_float)]


TM_FMT_MAX = 48


class TmCsvMapping(ctypes.Structure):
    _fields_ = [("col_timestamp", ctypes.c_int32), ("col_src_bank", ctypes.c_int32),
                ("col_src_account", ctypes.c_int32), ("col_dst_bank", ctypes.c_int32),
                ("col_dst_account", ctypes.c_int32), ("col_amount", ctypes.c_int32),
                ("col_currency", ctypes.c_int32), ("col_label", ctypes.c_int32),
                ("needed", ctypes.c_int32), ("delimiter", ctypes.c_int32),
                ("tick_seconds", ctypes.c_int64), ("n_fmt", ctypes.c_int32),
                ("fmt_op", ctypes.c_int32 * TM_FMT_MAX), ("fmt_arg", ctypes.c_int32 * TM_FMT_MAX)]


class TmIngestInfo(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("n_edges", ctypes.c_int64), ("n_nodes", ctypes.c_int64),
                ("n_currency", ctypes.c_int64), ("err_row", ctypes.c_int64), ("err_status", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("err_begin", ctypes.c_int64), ("err_end", ctypes.c_int64)]


class TmMineStats(ctypes.Structure):
    _fields_ = [("triggers", ctypes.c_int64), ("heavy_triggers", ctypes.c_int64),
                ("kernel_launches", ctypes.c_int64), ("light_ms", ctypes.c_float),
                ("heavy_ms", ctypes.c_float), ("total_ms", ctypes.c_float),
                ("prep_ms", ctypes.c_float)]


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
    "tm_mine_prepare": (ctypes.c_int, [_P, ctypes.POINTER(TmPlanDesc), ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, _P]),
    "tm_mine_release": (ctypes.c_int, [_P]),
    "tm_mine_members": (ctypes.c_int, [_P, ctypes.POINTER(TmPlanDesc), ctypes.c_int, ctypes.c_int64,
                                       ctypes.c_int64, _P, ctypes.c_int, _P]),
    "tm_last_mine_stats": (ctypes.c_int, [_P, ctypes.POINTER(TmMineStats)]),
    "tm_csv_format": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.c_int, _P, ctypes.POINTER(ctypes.c_int64)]),
    "tm_csv_fetch": (ctypes.c_int, [_P, _P, ctypes.c_int64]),
    "tm_collect_instances": (ctypes.c_int, [_P, ctypes.POINTER(TmPlanDesc), ctypes.c_int, ctypes.c_int64,
                                            ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "tm_fetch_instances": (ctypes.c_int, [_P, _P, ctypes.c_int64]),
    "tm_graph_set_attrs": (ctypes.c_int, [_P, _P, _P, ctypes.c_int32, _P]),
    "tm_vm_mine": (ctypes.c_int, [_P, ctypes.POINTER(TmVmProgram), ctypes.c_int64, ctypes.c_int64, _P]),
    "tm_vm_collect": (ctypes.c_int, [_P, ctypes.POINTER(TmVmProgram), ctypes.c_int32, ctypes.c_int64,
                                     ctypes.c_int64, ctypes.POINTER(ctypes.c_int64)]),
    "tm_vm_members": (ctypes.c_int, [_P, ctypes.POINTER(TmVmProgram), ctypes.c_int64, ctypes.c_int64, _P]),
    "tm_ingest_csv": (ctypes.c_int, [ctypes.c_int, _P, ctypes.c_int64, ctypes.c_int, ctypes.POINTER(TmCsvMapping),
                                     _P, ctypes.POINTER(_P), ctypes.POINTER(TmIngestInfo)]),
    "tm_ingest_fetch": (ctypes.c_int, [_P, _P, _P, _P, _P, _P, _P]),
    "tm_ingest_vocab": (ctypes.c_int, [_P, _P, _P, ctypes.c_int64]),
    "tm_ingest_graph": (ctypes.c_int, [_P, ctypes.POINTER(_P)]),
    "tm_ingest_free": (None, [_P]),
    "tm_set_profiling": (ctypes.c_int, [_P, ctypes.c_int]),
    "tm_kernel_launch_count": (ctypes.c_int64, []),
    "tm_host_alloc": (ctypes.c_int, [ctypes.c_int64, ctypes.POINTER(_P)]),
    "tm_host_free": (None, [_P]),
    "tm_last_error": (ctypes.c_char_p, []),
    "tm_graph_free": (None, [_P]),
}
ABI_VERSION = 7

# work counters of -DTM_COUNTERS=1 builds (tm_debug_counters; order of
# dev::CtrId in csrc/tm_device.cuh)
COUNTER_NAMES = ["trig", "u_walk", "u_item", "v_walk", "v_item", "window", "bisect32", "scan_call",
                 "scan_load", "pair_call", "bisect64", "inner_call", "inner_walk", "chain1", "chain2",
                 "chain3", "chain4", "close_call", "close_walk", "dom_task", "chain_task", "first",
                 "inner_skip", "pulls", "queue_full", "slot_full", "useful_over", "bloom_over",
                 "chain_over"]


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
