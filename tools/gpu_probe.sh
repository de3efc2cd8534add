cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.log
for rw in 4 8 4 8; do KGE_ROW_WARPS=$rw timeout 600 python bench.py --steps 3000 --warmup 50 --no-cpu-baseline --e2e-steps 500 > gpurun_out/bench_rw$rw.log 2>&1; python - <<'PY' >> gpurun_out/rw_ab.txt
import json, os
rw = os.environ.get("RW")
PY
grep '^{' gpurun_out/bench_rw$rw.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rw=$rw', round(d['value']/1e6,3), round(d['ms_per_step']*1e3,2), round(d['e2e']['value']/1e6,3))" >> gpurun_out/rw_ab.txt; done
