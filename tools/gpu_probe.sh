cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 120 ./tools/tmem_probe > gpurun_out/tmem_probe.txt 2>&1
