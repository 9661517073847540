# round-2 final evidence (after deferral, stored task windows, fill shape)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02v_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/r02v_gpu_tests.log 2>&1
timeout 1500 python bench.py > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r02v_launches_hl.csv $B > gpurun_out/r02v_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp|k_mine_chains|k_mine_tasks" -c 4 \
   -o gpurun_out/r02v_prof_hl $B > gpurun_out/r02v_full.log 2>&1
timeout 1500 python tools/emulate_ranks.py hi-large > gpurun_out/r02v_emulate.jsonl 2> gpurun_out/r02v_emulate.err
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02v_launches_rank8.csv \
   python tools/emulate_ranks.py hi-large --worlds 8 --reps 1 > gpurun_out/r02v_emulate8_ncu.log 2>&1
timeout 2400 python tools/sweep_cycles.py hi-medium --deltas 604800 --lengths 8 --reps 0 --budget 3000 --parity-blocks 8 --parity-block 100 > gpurun_out/r02v_sweep_c8.jsonl 2> gpurun_out/r02v_sweep_c8.err
