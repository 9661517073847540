# A/B: rolled short per-column loops in the trigger kernel (TM_WARM_ROLL) on top of the cold-path shrink
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/cold1p.so ablibs/warm.so ablibs/base.so ablibs/cold1p.so ablibs/warm.so >> gpurun_out/r02ao_ab.jsonl 2>> gpurun_out/r02ao_ab.err
done
