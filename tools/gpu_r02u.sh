set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_libs.py hi-large ablibs/tw.so ablibs/f1024x2.so ablibs/f256x8.so ablibs/f1024x4.so > gpurun_out/r02u_ab.jsonl 2> gpurun_out/r02u_ab.err
