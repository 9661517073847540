set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02aa_gpu_tests.log 2>&1
for cfg in hi-large hi-medium hi-small; do
  timeout 900 python tools/ab_libs.py $cfg ablibs/final.so ablibs/tsplit.so >> gpurun_out/r02aa_ab.jsonl 2>> gpurun_out/r02aa_ab.err
done
