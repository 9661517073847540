# final commit: GPU suite, smoke, default bench, reference arm, launch list (+DRAM bytes)
set -x
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/fin2_tests.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin2_smoke.txt 2>&1
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
   --log-file gpurun_out/fin2_launches_hl.csv $B > gpurun_out/fin2_launch.log 2>&1
python tools/launch_list.py gpurun_out/fin2_launches_hl.csv --config hi-large --md gpurun_out/fin2_launches_hl.md > gpurun_out/fin2_launch_summary.txt 2>&1
cp profiles/ncu_traffic.json gpurun_out/fin2_ncu_traffic.json
timeout 1500 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/fin2_ref.json 2> gpurun_out/fin2_ref.err
