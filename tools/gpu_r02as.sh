# A/B: window scan-vs-probe threshold (TM_SCAN_WIN 8 / 16 / 32) at the final code
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/scan8.so ablibs/scan32.so ablibs/base.so ablibs/scan8.so ablibs/scan32.so >> gpurun_out/r02as_ab.jsonl 2>> gpurun_out/r02as_ab.err
done
