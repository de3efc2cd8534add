#!/bin/bash
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/gpu_iter.sh
timeout 300 python tools/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1
