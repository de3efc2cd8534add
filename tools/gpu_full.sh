#!/bin/bash
# Round evidence: build, GPU tests, smoke, default bench, per-config benches, launch list, ncu --set full
# (application replay, caches as the step leaves them) of the step kernels on the bench workload, steady trace.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.log 2>&1
bash tools/gpu_configs.sh
timeout 300 python tools/trace_step.py freebase steady > gpurun_out/trace_steady.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_ -s 400 -c 200 --csv \
  --log-file gpurun_out/launches.csv python tools/ncu_step.py freebase 500 > gpurun_out/ncu_launch.log 2>&1
timeout 2400 ncu --set full --clock-control none --cache-control none --import-source on --replay-mode application \
  -k regex:"k_tc_fwd|k_tc_bwd|k_update|k_gather" -s 200 -c 4 -o gpurun_out/prof_fb \
  python tools/ncu_step.py freebase 210 > gpurun_out/ncu_full.log 2>&1
echo done
