"""Build recipe for libtempmine_b200.so (sm_100a, in-tree).

`python -m paper_2604_12241_b200.build` or `build()` from __graft_entry__.
nvcc compiles each .cu for `-gencode arch=compute_100a,code=sm_100a` with
-lineinfo and links one shared library next to this file; the library only
depends on the CUDA runtime (static) — no torch symbols cross the C ABI.
"""

from __future__ import annotations

import os
import shutil
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

HERE = Path(__file__).resolve().parent
CSRC = HERE / "csrc"
LIB = HERE / "libtempmine_b200.so"
# test-only variant: tiny queue / split / backward-set / Bloom-list caps and
# work counters, so the parity suite drives every exactness-preserving
# fallback path (tests/test_gpu_fallbacks.py); never loaded by the package
TINY_LIB = HERE / "libtempmine_b200_tinycaps.so"
TINY_DEFINES = ("TM_TASK_CAP=64", "TM_SPLIT_CAP=8", "TM_BCAP=3", "TM_BLOOM_LIST=8", "TM_CHAIN_CAP=16",
                "TM_COUNTERS=1")
SOURCES = ["tm_api.cu", "tm_sort.cu", "tm_graph.cu", "tm_slab.cu", "tm_mine.cu", "tm_members.cu", "tm_export.cu", "tm_instances.cu", "tm_vm.cu", "tm_ingest.cu"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def needs_build() -> bool:
    if not LIB.exists():
        return True
    mtime = LIB.stat().st_mtime
    deps = [CSRC / s for s in SOURCES] + list(CSRC.glob("*.cuh")) + [HERE.parent / "include" / "tempmine_b200.h"]
    return any(d.stat().st_mtime > mtime for d in deps)


def build(force: bool = False, verbose: bool = False, defines=(), out: Path | None = None) -> Path:
    """Compile the library; `defines` (e.g. ["TM_SMALL_RUN=0"]) and `out` build tuning variants."""
    if not force and not needs_build() and not defines and out is None:
        return LIB
    objdir = HERE / "build" / ("_".join(d.replace("=", "") for d in defines) or "default")
    objdir.mkdir(parents=True, exist_ok=True)
    flags = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
             "--expt-relaxed-constexpr", *ARCH, *[f"-D{d}" for d in defines]]

    def compile_one(src: str) -> str:
        obj = objdir / (Path(src).stem + ".o")
        cmd = [nvcc(), "-c", str(CSRC / src), "-o", str(obj), *flags]
        res = subprocess.run(cmd, capture_output=True, text=True)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{res.stderr}")
        if verbose and res.stderr:
            print(res.stderr, file=sys.stderr)
        return str(obj)

    with ThreadPoolExecutor(max_workers=min(len(SOURCES), os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, SOURCES))
    target = out or LIB
    tmp = target.with_suffix(".so.tmp")
    cmd = [nvcc(), "-shared", "-o", str(tmp), *objs, *ARCH, "-cudart", "static"]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        raise RuntimeError(f"link failed:\n{res.stderr}")
    os.replace(tmp, target)
    return target


def build_tiny(force: bool = False) -> Path:
    """The tiny-caps test variant (TINY_DEFINES) next to the product library."""
    if not force and TINY_LIB.exists() and LIB.exists() and TINY_LIB.stat().st_mtime >= LIB.stat().st_mtime:
        return TINY_LIB
    return build(force=True, defines=TINY_DEFINES, out=TINY_LIB)


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--tiny" in sys.argv:
        print(build_tiny(force=True))
