# final code at the other BASELINE shapes (bench lines, with sampled-block parity)
set -x
mkdir -p gpurun_out
timeout 900 python bench.py --config hi-medium > gpurun_out/shape_hi-medium.json 2> gpurun_out/shape_hi-medium.err
timeout 900 python bench.py --config hi-small > gpurun_out/shape_hi-small.json 2> gpurun_out/shape_hi-small.err
