#!/bin/bash
# Round evidence: build, full GPU tests, smoke, default bench (+ reference arm), every config, launch lists of the
# Freebase step and the TransR step. Everything lands in gpurun_out/.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -q -m gpu -rfE --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
bash tools/gpu_configs.sh
timeout 600 python bench.py --precision bf16 --steps 20000 --warmup 50 --no-cpu-baseline --e2e-steps 1000 > gpurun_out/bench_bf16.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 400 -c 200 --csv \
  --log-file gpurun_out/launches_freebase.csv python tools/ncu_step.py freebase 500 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 200 -c 120 --csv \
  --log-file gpurun_out/launches_transr.csv python tools/ncu_step.py fb15k 260 transr 200 > gpurun_out/ncu_launch_tr.log 2>&1
echo done
