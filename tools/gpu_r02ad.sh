# A/B: full-row staging (TM_STAGE_ALL) vs base; e2e phase diagnosis at HI-Large
set -x
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py hi-large ablibs/base.so ablibs/stageall.so ablibs/base.so ablibs/stageall.so > gpurun_out/r02ad_ab.jsonl 2> gpurun_out/r02ad_ab.err
timeout 900 python tools/diag_e2e.py hi-large 12 > gpurun_out/r02ad_e2e.txt 2>&1
