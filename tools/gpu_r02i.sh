# runtime chain depth (smaller code) + short-run off: parity; A/B joint 4-window bisection
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02i_gpu_tests.log 2>&1
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/win4.so > gpurun_out/r02i_ab.jsonl 2> gpurun_out/r02i_ab.err
timeout 900 python tools/ab_libs.py hi-small ablibs/base.so ablibs/win4.so >> gpurun_out/r02i_ab.jsonl 2>> gpurun_out/r02i_ab.err
timeout 900 python tools/ab_libs.py hi-medium ablibs/base.so ablibs/win4.so >> gpurun_out/r02i_ab.jsonl 2>> gpurun_out/r02i_ab.err
