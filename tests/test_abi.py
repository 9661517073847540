"""The C-ABI library builds for sm_100a, loads, and exports every symbol the
header declares (no compute calls: this runs without a GPU)."""

from __future__ import annotations

import ctypes
import re
import subprocess

from conftest import ROOT

HEADER = ROOT / "include" / "tempmine_b200.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(tm_[a-z_]+)\s*\(", text)))


def test_library_builds_and_loads():
    from paper_2604_12241_b200 import build, _lib
    path = build.build()
    assert path.exists()
    lib = _lib.load()
    assert lib.tm_abi_version() == _lib.ABI_VERSION


def test_exports_every_declared_symbol():
    from paper_2604_12241_b200 import _lib
    lib = ctypes.CDLL(str(_lib.LIB_PATH))
    syms = declared_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(lib, s), s
    # the wrapper binds exactly the declared surface
    assert sorted(_lib.SIGNATURES) == syms


def test_library_is_sm100a():
    from paper_2604_12241_b200 import _lib
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


def test_plan_desc_layout_matches_header():
    from paper_2604_12241_b200 import _lib
    assert ctypes.sizeof(_lib.TmPlanDesc) == 32
    assert _lib.TmPlanDesc.delta.offset == 24


def test_missing_library_fails_loudly(tmp_path):
    import pytest
    from paper_2604_12241_b200 import _lib
    saved = _lib._lib
    try:
        _lib._lib = None
        with pytest.raises(RuntimeError, match="no CPU fallback"):
            _lib.load(tmp_path / "absent.so")
    finally:
        _lib._lib = saved
