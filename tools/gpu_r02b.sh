# slab view: parity suite, then HI-Large / HI-Small A/B of the global vs slab view
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02b_gpu_tests.log 2>&1
for cfg in hi-small hi-large; do
  for sl in 0 1; do
    TM_SLABS=$sl timeout 900 python bench.py --config $cfg --steps 5 --warmup 2 --no-e2e --no-parity \
      > gpurun_out/r02b_bench_${cfg}_slab$sl.json 2> gpurun_out/r02b_bench_${cfg}_slab$sl.err
  done
done
