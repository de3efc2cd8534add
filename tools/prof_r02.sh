cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
python tools/trace_step.py freebase steady > gpurun_out/trace_steady.txt 2>&1
python tools/trace_step.py freebase > gpurun_out/trace_isolated.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 300 -c 80 --csv --log-file gpurun_out/r02_launches.csv python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/ncu_list.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_tc_fwd|k_tc_bwd|k_update|k_gather" -s 40 -c 4 -o gpurun_out/r02_full python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 20 > gpurun_out/ncu_full.log 2>&1
echo done
