#!/bin/bash
# bench lines for every BASELINE.json config on one GPU (the default bench is configs[4], Freebase TransE-L2)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
run() { echo "== $*"; timeout 600 python bench.py --steps 2000 --warmup 20 --e2e-steps 500 "$@" 2>&1 | grep '^{' ; }
{
run --workload tiny
run --workload fb15k --model distmult
run --workload fb15k --model complex
run --workload fb15k --model distmult --precision fp32
run --workload wn18 --model rotate
run --workload wn18 --model transe_l1
run --workload fb15k_transr
run --workload freebase --precision fp32
} > gpurun_out/configs.log 2>&1
