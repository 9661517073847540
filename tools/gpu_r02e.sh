# slab view without own-window tables; ncu of the warp kernel in the slab view
set -x
mkdir -p gpurun_out
B="python bench.py --config hi-large --steps 3 --warmup 2 --no-e2e --no-parity --no-families"
for own in 0 1; do
  TM_SLABS=1 TM_OWN=$own timeout 900 $B > gpurun_out/r02e_bench_own$own.json 2> gpurun_out/r02e_bench_own$own.err
done
TM_SLABS=1 TM_OWN=0 timeout 1200 ncu --set full --clock-control none --import-source on \
   -k regex:"k_mine_warp|k_mine_tasks" -c 3 -o gpurun_out/r02e_prof_hl_slab1_own0 \
   python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families > gpurun_out/r02e_full.log 2>&1
