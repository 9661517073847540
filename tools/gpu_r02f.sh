# new slab build + slab-local hub probes: parity, then HI-Large / HI-Small step + launch list
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02f_gpu_tests.log 2>&1
for cfg in hi-small hi-large; do
  timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-parity > gpurun_out/r02f_bench_$cfg.json 2> gpurun_out/r02f_bench_$cfg.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02f_launches_hl.csv \
  python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02f_launch.log 2>&1
