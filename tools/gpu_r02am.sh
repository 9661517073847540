# A/B: slab of a rank from shared-memory slab starts in the view build (TM_SLAB_SEARCH)
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py hi-large ablibs/base.so ablibs/search.so ablibs/base.so ablibs/search.so > gpurun_out/r02am_ab.jsonl 2> gpurun_out/r02am_ab.err
TM_LIB=$PWD/ablibs/search.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -x -q > gpurun_out/r02am_tests.txt 2>&1
