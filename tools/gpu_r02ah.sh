# full GPU suite + bench on the lane-list / one-group build
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02ah_tests.txt 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02ah_smoke.txt 2>&1
timeout 1500 python bench.py > gpurun_out/r02ah_bench.json 2> gpurun_out/r02ah_bench.err
