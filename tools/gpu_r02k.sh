# vector-load short runs / window scans: parity + A/B; e2e phase diagnostics
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r02k_gpu_tests.log 2>&1
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/novec.so ablibs/vecrun.so ablibs/vecscan.so > gpurun_out/r02k_ab.jsonl 2> gpurun_out/r02k_ab.err
timeout 900 python tools/ab_libs.py hi-small ablibs/base.so ablibs/novec.so >> gpurun_out/r02k_ab.jsonl 2>> gpurun_out/r02k_ab.err
timeout 900 python tools/diag_e2e.py hi-large 6 > gpurun_out/r02k_diag_e2e.txt 2>&1
