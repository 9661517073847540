set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt 2>&1
free -g > gpurun_out/r02a_free.txt; nproc >> gpurun_out/r02a_free.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02a_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02a_launches_hl.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02a_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_mine|k_own|k_lo_table" -c 12 -o gpurun_out/r02a_prof_hl python bench.py --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02a_ncu_full.log 2>&1
ls -la gpurun_out | tail -20
