# prepared views / contiguous pieces: GPU tests; rank emulation; TMA + slab-width A/B
set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02o_gpu_tests.log 2>&1
timeout 1500 python tools/ab_libs.py hi-large ablibs/base.so ablibs/tma.so > gpurun_out/r02o_ab.jsonl 2> gpurun_out/r02o_ab.err
TM_SLAB_WMULT=2 timeout 900 python tools/ab_libs.py hi-large ablibs/base.so >> gpurun_out/r02o_ab.jsonl 2>> gpurun_out/r02o_ab.err
timeout 1500 python tools/emulate_ranks.py hi-large > gpurun_out/r02o_emulate.jsonl 2> gpurun_out/r02o_emulate.err
timeout 900 python tools/work_profile.py ablibs/ctr.so hi-large > gpurun_out/r02o_work.txt 2>&1
TM_CARVEOUT=35 timeout 900 python tools/ab_libs.py hi-large ablibs/base.so >> gpurun_out/r02o_ab.jsonl 2>> gpurun_out/r02o_ab.err
TM_CARVEOUT=60 timeout 900 python tools/ab_libs.py hi-large ablibs/base.so >> gpurun_out/r02o_ab.jsonl 2>> gpurun_out/r02o_ab.err
