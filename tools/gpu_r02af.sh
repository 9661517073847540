# A/B: packed lane-column lists (TM_LANE_DESC) and shared-trip bisection (TM_WIN_FIXED)
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/nolane.so ablibs/lane.so ablibs/fixed.so ablibs/nolane.so ablibs/lane.so ablibs/fixed.so >> gpurun_out/r02af_ab.jsonl 2>> gpurun_out/r02af_ab.err
done
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/r02af_parity.txt 2>&1
