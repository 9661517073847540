# final confirmation: smoke, A/B of the final library, default bench
set -x
mkdir -p gpurun_out
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02z_smoke.txt 2>&1
for cfg in hi-large hi-medium hi-small; do
  timeout 900 python tools/ab_libs.py $cfg ablibs/final.so >> gpurun_out/r02z_ab.jsonl 2>> gpurun_out/r02z_ab.err
done
timeout 1500 python bench.py > gpurun_out/r02z_bench.json 2> gpurun_out/r02z_bench.err
