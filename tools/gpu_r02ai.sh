# A/B per-entry slots; launch list (+DRAM bytes) of one HI-Large call; ncu --set full of the task kernels
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py hi-large ablibs/lanes1.so ablibs/slots.so ablibs/lanes1.so ablibs/slots.so > gpurun_out/r02ai_ab.jsonl 2> gpurun_out/r02ai_ab.err
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/r02ai_launches_hl.csv $B > gpurun_out/r02ai_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_tasks|k_mine_chains|k_slab_fill" -c 8 \
   -o gpurun_out/r02ai_prof_tasks $B > gpurun_out/r02ai_full.log 2>&1
