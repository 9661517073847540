# A/B: owner / (nbr, prev) loads hoisted next to the rank loads in the slab view build
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py hi-large ablibs/base.so ablibs/hoist.so ablibs/hoist2.so ablibs/base.so ablibs/hoist.so ablibs/hoist2.so > gpurun_out/r02ap_ab.jsonl 2> gpurun_out/r02ap_ab.err
TM_LIB=$PWD/ablibs/hoist2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/r02ap_tests.txt 2>&1
