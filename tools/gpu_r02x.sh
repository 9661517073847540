# long-window rule: tests (fallbacks incl. short-window deferral), 3 d / 7 d sweep cells, HI-Large call
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02x_gpu_tests.log 2>&1
timeout 900 python tools/ab_libs.py hi-large paper_2604_12241_b200/libtempmine_b200.so > gpurun_out/r02x_ab.jsonl 2> gpurun_out/r02x_ab.err
timeout 2400 python tools/sweep_cycles.py hi-medium --deltas 259200,604800 --lengths 4,5,6,7 --budget 200 --reps 1 > gpurun_out/r02x_sweep.jsonl 2> gpurun_out/r02x_sweep.err
