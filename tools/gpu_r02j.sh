set -x
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02j_launches_hl.csv \
  python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02j_launch.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp|k_mine_tasks|k_slab_fill|k_slab_edges" -c 5 \
  -o gpurun_out/r02j_prof_hl python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02j_full.log 2>&1
