#!/bin/bash
# k_tr_dm_tc timing by epilogue mode (KGE_TR_DM_MODE: 0 full, 1 no M update, 2 no epilogue) -- timing only
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 1 2; do
  KGE_TR_DM_MODE=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tr_dm_tc -s 5 -c 5 --csv --log-file gpurun_out/dm_$m.csv python bench.py --workload fb15k_transr --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 5 > /dev/null 2>&1
done
echo done
