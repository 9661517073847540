# A/B: warp-cooperative bisection of long trigger runs (TM_COOP_RUN)
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/coop32.so ablibs/coop64.so ablibs/coop128.so ablibs/coop256.so ablibs/base.so ablibs/coop64.so >> gpurun_out/r02aj_ab.jsonl 2>> gpurun_out/r02aj_ab.err
done
