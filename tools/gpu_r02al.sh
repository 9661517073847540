# A/B: packed per-lane trigger context records in WarpShared (TM_WS_PACK)
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium hi-small; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/pack.so ablibs/base.so ablibs/pack.so >> gpurun_out/r02al_ab.jsonl 2>> gpurun_out/r02al_ab.err
done
