"""ctypes wrapper of oracle/libtm_oracle.so — TEST INFRASTRUCTURE ONLY.

The C file restates the reference column semantics (kernels.py:290-402,
engine.py:516-562 on SURVEY.md Appendix B); this wrapper only marshals
arrays.  Pinned to the reference by tests/test_oracle_golden.py.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "libtm_oracle.so"

# base column name -> (family, endpoint, direction, exclude_trigger, cycle_len, default min_size)
# family codes: 1 FAN, 2 DEGREE, 3 CYCLE, 4 SG, 5 GS, 6 STACK
COLUMN_FAMILIES = {
    "fan_in": (1, 1, 0, 1, 0, 1), "fan_out": (1, 0, 1, 1, 0, 1),
    "deg_in_src": (2, 0, 0, 0, 0, 1), "deg_out_src": (2, 0, 1, 0, 0, 1),
    "deg_in_dst": (2, 1, 0, 0, 0, 1), "deg_out_dst": (2, 1, 1, 0, 0, 1),
    "cycle_2": (3, 0, 0, 0, 2, 1), "cycle_3": (3, 0, 0, 0, 3, 1), "cycle_4": (3, 0, 0, 0, 4, 1),
    "cycle_5": (3, 0, 0, 0, 5, 1), "cycle_6": (3, 0, 0, 0, 6, 1), "cycle_7": (3, 0, 0, 0, 7, 1),
    "cycle_8": (3, 0, 0, 0, 8, 1),
    "sg_count": (4, 0, 0, 0, 0, 2), "gs_count": (5, 0, 0, 0, 0, 2), "stack_count": (6, 0, 0, 0, 0, 1),
}


class OgPlan(ctypes.Structure):
    _fields_ = [("family", ctypes.c_int32), ("endpoint", ctypes.c_int32),
                ("direction", ctypes.c_int32), ("exclude_trigger", ctypes.c_int32),
                ("cycle_len", ctypes.c_int32), ("min_size", ctypes.c_int32),
                ("delta", ctypes.c_int64)]


_lib = None


def load() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        if not LIB.exists() or LIB.stat().st_mtime < (HERE / "tm_oracle.c").stat().st_mtime:
            subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
        lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        lib.og_build.restype = P
        lib.og_build.argtypes = [ctypes.c_int64, ctypes.c_int64, P, P, P]
        lib.og_free.argtypes = [P]
        lib.og_export.argtypes = [P, ctypes.c_int, P, P, P, P]
        lib.og_mine.restype = ctypes.c_int
        lib.og_mine.argtypes = [P, ctypes.POINTER(OgPlan), ctypes.c_int, ctypes.c_int64,
                                ctypes.c_int64, P, ctypes.c_int]
        _lib = lib
    return _lib


def column(base: str, delta: int, min_size: int | None = None) -> tuple:
    fam, ep, dr, ex, cl, k0 = COLUMN_FAMILIES[base]
    return (fam, ep, dr, ex, cl, k0 if min_size is None else int(min_size), int(delta))


class OracleGraph:
    def __init__(self, src, dst, time, node_count: int | None = None):
        self.src = np.ascontiguousarray(src, dtype=np.int64)
        self.dst = np.ascontiguousarray(dst, dtype=np.int64)
        self.time = np.ascontiguousarray(time, dtype=np.int64)
        if node_count is None:
            node_count = int(max(self.src.max(), self.dst.max())) + 1 if len(self.src) else 0
        self.node_count = int(node_count)
        self.edge_count = len(self.src)
        self._h = load().og_build(self.node_count, self.edge_count, self.src.ctypes.data,
                                  self.dst.ctypes.data, self.time.ctypes.data)
        if not self._h:
            raise MemoryError("og_build failed")

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.og_free(self._h)
            self._h = None

    def export(self, direction: str):
        d = 1 if direction == "out" else 0
        out = [np.empty(self.node_count + 1, np.int64)] + [np.empty(self.edge_count, np.int64) for _ in range(3)]
        load().og_export(self._h, d, *[a.ctypes.data for a in out])
        return tuple(out)

    def mine(self, columns: list[tuple], lo: int = 0, hi: int | None = None,
             threads: int | None = None) -> np.ndarray:
        hi = self.edge_count if hi is None else hi
        arr = (OgPlan * max(len(columns), 1))(*[OgPlan(*c) for c in columns])
        out = np.empty((hi - lo, len(columns)), dtype=np.int64)
        rc = load().og_mine(self._h, arr, len(columns), lo, hi, out.ctypes.data,
                            threads or os.cpu_count() or 1)
        if rc != 0:
            raise RuntimeError(f"og_mine failed ({rc})")
        return out
