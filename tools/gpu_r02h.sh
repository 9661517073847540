# short-run windows + register-resident slab fill: parity, launch list, short-run A/B
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02h_gpu_tests.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02h_launches_hl.csv \
  python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02h_launch.log 2>&1
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/sr0.so ablibs/sr8.so > gpurun_out/r02h_ab.jsonl 2> gpurun_out/r02h_ab.err
timeout 900 python tools/ab_libs.py hi-small ablibs/base.so ablibs/sr0.so ablibs/sr8.so >> gpurun_out/r02h_ab.jsonl 2>> gpurun_out/r02h_ab.err
