# A/B: cold-path code out of the trigger kernel's instruction footprint (#pragma unroll 1 on
# the queue-full / emission / permuted-row loops; emission out of line)
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium hi-small; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/cold1.so ablibs/cold2.so ablibs/base.so ablibs/cold1.so ablibs/cold2.so >> gpurun_out/r02an_ab.jsonl 2>> gpurun_out/r02an_ab.err
done
