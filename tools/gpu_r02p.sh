# slab-view rule + cheap restricted prep: tests (both views), rank emulation, benches
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02p_gpu_tests.log 2>&1
timeout 1500 python tools/emulate_ranks.py hi-large > gpurun_out/r02p_emulate.jsonl 2> gpurun_out/r02p_emulate.err
for cfg in hi-small hi-medium; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 --no-e2e --no-parity > gpurun_out/r02p_bench_$cfg.json 2> gpurun_out/r02p_bench_$cfg.err
done
