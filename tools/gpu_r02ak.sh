# A/B: flat_for item owners by ballot (TM_FLAT_BALLOT)
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium hi-small; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/ballot.so ablibs/base.so ablibs/ballot.so >> gpurun_out/r02ak_ab.jsonl 2>> gpurun_out/r02ak_ab.err
done
