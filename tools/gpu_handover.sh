#!/bin/bash
# hand-over experiments: steady-step trace with/without the next-step row prefetch and with smaller entity tables
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/trace_step.py freebase steady > gpurun_out/ho_default.txt 2>&1
KGE_NO_PREFETCH=1 timeout 300 python tools/trace_step.py freebase steady > gpurun_out/ho_noprefetch.txt 2>&1
KGE_TRACE_NE=8000000 timeout 300 python tools/trace_step.py freebase steady > gpurun_out/ho_8M.txt 2>&1
KGE_TRACE_NE=1000000 timeout 300 python tools/trace_step.py freebase steady > gpurun_out/ho_1M.txt 2>&1
KGE_TRACE_NE=50000 timeout 300 python tools/trace_step.py freebase steady > gpurun_out/ho_50k.txt 2>&1
echo done
