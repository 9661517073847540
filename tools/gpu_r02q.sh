# round-2 evidence: default bench, launch list with DRAM, ncu full, reference arm, cycle_8 @ 7 d
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02q_smi.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r02q_bench.json 2> gpurun_out/r02q_bench.err
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r02q_launches_hl.csv $B > gpurun_out/r02q_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp|k_mine_tasks|k_slab_fill|k_slab_edges|k_slab_tile" -c 8 \
   -o gpurun_out/r02q_prof_hl $B > gpurun_out/r02q_full.log 2>&1
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/r02q_ref.json 2> gpurun_out/r02q_ref.err
timeout 1800 python tools/sweep_cycles.py hi-medium --deltas 604800 --lengths 8 --reps 0 --budget 3000 --parity-blocks 8 --parity-block 100 > gpurun_out/r02q_sweep_c8.jsonl 2> gpurun_out/r02q_sweep_c8.err
