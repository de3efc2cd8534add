#!/bin/bash
# round-2 GPU iteration: build, the given pytest selection (default: everything -m gpu), smoke, optional bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
SEL=${SEL:-tests}
timeout ${PYT_TIMEOUT:-2400} python -m pytest $SEL -q -m gpu -rfE --durations=25 ${PYT_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
if [ -n "$SMOKE" ]; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; fi
if [ -n "$BENCH" ]; then timeout 900 python bench.py $BENCH > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log; fi
echo done
