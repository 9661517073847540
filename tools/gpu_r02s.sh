# evidence with deferral: bench, launch list + DRAM, ncu full of k_mine_warp / chains / tasks, lines, ranks, e2e phases
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02s_smi.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r02s_bench.json 2> gpurun_out/r02s_bench.err
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r02s_launches_hl.csv $B > gpurun_out/r02s_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp|k_mine_chains|k_mine_tasks" -c 4 \
   -o gpurun_out/r02s_prof_hl $B > gpurun_out/r02s_full.log 2>&1
timeout 1500 python tools/emulate_ranks.py hi-large > gpurun_out/r02s_emulate.jsonl 2> gpurun_out/r02s_emulate.err
timeout 900 python tools/diag_e2e.py hi-large 5 > gpurun_out/r02s_diag_e2e.txt 2>&1
