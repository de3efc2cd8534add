#!/bin/bash
# One gpurun call: per-CTA trace of a step + ncu --set full (application replay) of the step kernels on Freebase.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/trace_step.py freebase > gpurun_out/trace.log 2>&1
timeout 2400 ncu --set full --clock-control none --import-source on --replay-mode application \
  -k regex:"k_tc_fwd|k_tc_bwd|k_update|k_gather" -s 200 -c 4 -o gpurun_out/prof_fb \
  python tools/ncu_step.py freebase 210 > gpurun_out/ncu_full.log 2>&1
echo done
