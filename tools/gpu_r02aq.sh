# A/B: trigger-kernel register cap 40 (TM_WARP_MINB_DEFER 22 / 24) after the footprint cut
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/minb22.so ablibs/minb24.so ablibs/base.so ablibs/minb22.so ablibs/minb24.so >> gpurun_out/r02aq_ab.jsonl 2>> gpurun_out/r02aq_ab.err
done
