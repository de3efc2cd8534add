#!/bin/bash
# gather -> forward hand-over experiment: steady trace and device bench with / without KGE_GATHER_FENCE
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 python tools/trace_step.py freebase steady > gpurun_out/fence0.txt 2>&1
KGE_GATHER_FENCE=1 timeout 300 python tools/trace_step.py freebase steady > gpurun_out/fence1.txt 2>&1
timeout 600 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline --e2e-steps 200 > gpurun_out/bench0.log 2>&1
KGE_GATHER_FENCE=1 timeout 600 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline --e2e-steps 200 > gpurun_out/bench1.log 2>&1
echo done
