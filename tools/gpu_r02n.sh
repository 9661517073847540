set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/deep2.so ablibs/deep4.so ablibs/deep16.so ablibs/dom64.so ablibs/dom256.so > gpurun_out/r02n_ab.jsonl 2> gpurun_out/r02n_ab.err
timeout 2400 python tools/sweep_cycles.py hi-medium --budget 200 --reps 2 > gpurun_out/r02n_sweep.jsonl 2> gpurun_out/r02n_sweep.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02n_launches_hl.csv \
  python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02n_launch.log 2>&1
