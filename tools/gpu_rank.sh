#!/bin/bash
# Link-prediction ranking: GPU tests, throughput of the 8-query batched kernel vs one query per CTA.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for m in transe_l2 distmult rotate; do
  for qb in 1 8; do KGE_RANK_QB=$qb timeout 300 python tools/rank_bench.py $m 2000 >> gpurun_out/rank_bench.log 2>&1; done
done
