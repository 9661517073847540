# HI-Large launch lists (global vs slab view) + full ncu of the mining kernels
set -x
mkdir -p gpurun_out
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
for sl in 0 1; do
  TM_SLABS=$sl timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
     --log-file gpurun_out/r02d_launches_hl_slab$sl.csv $B > gpurun_out/r02d_launch_slab$sl.log 2>&1
done
TM_SLABS=0 timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:"k_mine_warp|k_mine_tasks|k_own_windows" -c 6 -o gpurun_out/r02d_prof_hl_slab0 $B > gpurun_out/r02d_full.log 2>&1
ls -la gpurun_out | tail
