"""Build library variants for tools/ab_libs.py into ablibs/ (git-ignored,
travels with gpurun):  python tools/build_variants.py NAME=DEF[,DEF...] ..."""
import sys
from concurrent.futures import ThreadPoolExecutor
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2604_12241_b200 import build as b  # noqa: E402

OUT = Path(__file__).resolve().parents[1] / "ablibs"
OUT.mkdir(exist_ok=True)


def one(spec):
    name, defs = spec.split("=", 1)
    return b.build(force=True, defines=tuple(d for d in defs.split(",") if d), out=OUT / f"{name}.so")


with ThreadPoolExecutor(4) as ex:
    for p in ex.map(one, sys.argv[1:]):
        print(p)
