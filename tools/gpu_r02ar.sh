# A/B: one-group instances of the task / chain kernels
set -x
mkdir -p gpurun_out
for cfg in hi-large hi-medium; do
timeout 900 python tools/ab_libs.py $cfg ablibs/base.so ablibs/onetask.so ablibs/base.so ablibs/onetask.so >> gpurun_out/r02ar_ab.jsonl 2>> gpurun_out/r02ar_ab.err
done
TM_LIB=$PWD/ablibs/onetask.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fallbacks.py -m gpu -x -q > gpurun_out/r02ar_tests.txt 2>&1
