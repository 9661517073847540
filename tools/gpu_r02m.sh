set -x
mkdir -p gpurun_out
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/ninner.so ablibs/nprobe.so ablibs/nboth.so ablibs/ptr2.so > gpurun_out/r02m_ab.jsonl 2> gpurun_out/r02m_ab.err
timeout 900 python tools/ab_libs.py hi-small ablibs/base.so ablibs/ninner.so ablibs/nprobe.so ablibs/nboth.so ablibs/ptr2.so >> gpurun_out/r02m_ab.jsonl 2>> gpurun_out/r02m_ab.err
timeout 1500 python tools/ref_python_bench.py hi-large --blocks 64 > gpurun_out/r02m_refpy_hl.json 2> gpurun_out/r02m_refpy_hl.err
