#!/bin/sh
# Stage the reference's Python package for oracle/ref_python.py (test
# infrastructure: bench.py's reference arm).  Copies the unmodified sources
# into oracle/_ref/ (git-ignored: not in history; NOT gpurun-ignored: it
# travels to the GPU box, where /root/reference does not exist).  A no-op
# when the reference is absent (the GPU box uses the staged copy).
set -e
HERE=$(cd "$(dirname "$0")" && pwd)
SRC=/root/reference/pkg/src/tempmine
[ -d "$SRC" ] || exit 0
mkdir -p "$HERE/_ref"
rm -rf "$HERE/_ref/tempmine"
cp -r "$SRC" "$HERE/_ref/tempmine"
find "$HERE/_ref/tempmine" -name __pycache__ -prune -exec rm -rf {} +
