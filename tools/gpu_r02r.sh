# deferred chain descents: parity suite (both views, fallbacks), A/B vs inline, register caps
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02r_gpu_tests.log 2>&1
for cfg in hi-large hi-medium hi-small; do
  timeout 900 python tools/ab_libs.py $cfg ablibs/defer.so ablibs/dmin24.so ablibs/dmin16.so ablibs/tminb2.so ablibs/tminb3.so >> gpurun_out/r02r_ab.jsonl 2>> gpurun_out/r02r_ab.err
  TM_DEFER=0 timeout 900 python tools/ab_libs.py $cfg ablibs/defer.so >> gpurun_out/r02r_ab_inline.jsonl 2>> gpurun_out/r02r_ab.err
done
