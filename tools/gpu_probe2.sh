cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tr|k_gather|k_update" -s 40 -c 40 --csv \
  --log-file gpurun_out/launches_tr.csv python tools/ncu_step.py fb15k 12 transr 200 > gpurun_out/ncu_tr.log 2>&1
