# round-2 final evidence: GPU suite, smoke, launch list (+DRAM bytes -> roofline.traffic), bench, ncu --set full
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_smi.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fin_tests.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.txt 2>&1
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/fin_launches_hl.csv $B > gpurun_out/fin_launch.log 2>&1
python tools/launch_list.py gpurun_out/fin_launches_hl.csv --config hi-large --md gpurun_out/fin_launches_hl.md > gpurun_out/fin_launch_summary.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/fin_ncu_traffic.json
timeout 1500 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp" -c 1 \
   -o gpurun_out/fin_prof_hl $B > gpurun_out/fin_full.log 2>&1
