# host topology, e2e with NUMA-local binding, ncu --set full of the trigger kernel (HI-Large)
set -x
mkdir -p gpurun_out
(nvidia-smi topo -m; lscpu; nproc; cat /proc/self/status | grep -i cpus_allowed_list; free -g) > gpurun_out/r02ae_topo.txt 2>&1
TM_BIND=1 timeout 900 python tools/diag_e2e.py hi-large 8 > gpurun_out/r02ae_e2e_bind.txt 2>&1
timeout 900 python tools/diag_e2e.py hi-large 8 > gpurun_out/r02ae_e2e_nobind.txt 2>&1
B="python bench.py --config hi-large --steps 1 --warmup 0 --no-e2e --no-parity --no-families"
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_mine_warp" -c 2 \
   -o gpurun_out/r02ae_prof_hl $B > gpurun_out/r02ae_full.log 2>&1
