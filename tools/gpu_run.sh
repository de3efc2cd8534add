#!/bin/bash
# One gpurun iteration: build, a pytest selection (SEL, default all -m gpu), then each ';;'-separated bench command line
# in BENCHES (python bench.py <args>, each with optional leading VAR=value env assignments) into gpurun_out/bench_<i>.log
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1; nproc >> gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ "${SEL}" != "none" ]; then
  timeout ${PYT_TIMEOUT:-2400} python -m pytest ${SEL:-tests} -q -m gpu -rfE --durations=15 ${PYT_ARGS} > gpurun_out/pytest_gpu.log 2>&1
  echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
fi
if [ -n "$SMOKE" ]; then timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; fi
i=0
IFS=';;' read -ra CMDS <<< "$BENCHES"
for c in "${CMDS[@]}"; do
  [ -z "${c// }" ] && continue
  i=$((i+1))
  echo "$c" > gpurun_out/bench_$i.log
  timeout ${BENCH_TIMEOUT:-900} env $c >> gpurun_out/bench_$i.log 2>&1
  echo "rc=$?" >> gpurun_out/bench_$i.log
done
echo done
