set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02t_gpu_tests.log 2>&1
for cfg in hi-large hi-medium hi-small; do
  timeout 900 python tools/ab_libs.py $cfg ablibs/defer.so ablibs/tw.so >> gpurun_out/r02t_ab.jsonl 2>> gpurun_out/r02t_ab.err
done
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r02t_launches_hl.csv python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02t_launch.log 2>&1
