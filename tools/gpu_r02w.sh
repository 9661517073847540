# onesweep scatter: tests, graph build timing; smaller shapes; full sweep with per-cell parity
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02w_gpu_tests.log 2>&1
timeout 900 python tools/diag_e2e.py hi-large 4 > gpurun_out/r02w_diag_e2e.txt 2>&1
for cfg in hi-small hi-medium; do
  timeout 900 python bench.py --config $cfg --steps 10 --warmup 3 > gpurun_out/r02w_bench_$cfg.json 2> gpurun_out/r02w_bench_$cfg.err
done
timeout 2700 python tools/sweep_cycles.py hi-medium --budget 200 --reps 2 --lengths 2,3,4,5,6,7 > gpurun_out/r02w_sweep.jsonl 2> gpurun_out/r02w_sweep.err
