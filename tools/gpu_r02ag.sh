# A/B: one-group kernel instance, direction selects (sel2), evict-first trigger I/O
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/noone.so ablibs/one.so ablibs/sel.so ablibs/stream.so ablibs/noone.so ablibs/one.so ablibs/sel.so ablibs/stream.so >> gpurun_out/r02ag_ab.jsonl 2>> gpurun_out/r02ag_ab.err
done
