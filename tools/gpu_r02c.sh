# re-entry: GPU tests, slab A/B, default bench (HI-Large) with parity
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02c_smi.txt 2>&1
lscpu > gpurun_out/r02c_lscpu.txt 2>&1; nproc >> gpurun_out/r02c_lscpu.txt; free -g >> gpurun_out/r02c_lscpu.txt
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r02c_gpu_tests.log 2>&1
for cfg in hi-small hi-large; do
  for sl in 0 1; do
    TM_SLABS=$sl timeout 900 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-parity \
      > gpurun_out/r02c_bench_${cfg}_slab$sl.json 2> gpurun_out/r02c_bench_${cfg}_slab$sl.err
  done
done
timeout 1200 python bench.py > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err
ls -la gpurun_out | tail -30
