set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02l_gpu_tests.log 2>&1
timeout 1500 python bench.py > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err
timeout 900 python tools/diag_e2e.py hi-large 5 > gpurun_out/r02l_diag_e2e.txt 2>&1
