#!/bin/bash
# TransR A/B: tests, then bench + launch list with the default and with $ABENV set
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -q -m gpu -k "transr or rescal" -x -rfE > gpurun_out/pt.txt 2>&1
for v in A B; do
  if [ $v = B ]; then export $ABENV; fi
  python bench.py --workload fb15k_transr --steps 300 --warmup 20 --no-cpu-baseline --e2e-steps 50 > gpurun_out/b_$v.txt 2>&1
  ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 60 --csv --log-file gpurun_out/tr_launches_$v.csv python bench.py --workload fb15k_transr --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 5 > /dev/null 2>&1
done
python - <<'PY'
import csv, collections
for v in "AB":
    rows=list(csv.reader(open(f'gpurun_out/tr_launches_{v}.csv')))
    hdr=None; d=collections.OrderedDict()
    for r in rows:
        if r and r[0]=='ID': hdr=r; continue
        if hdr and len(r)==len(hdr):
            x=dict(zip(hdr,r)); d.setdefault(x['Kernel Name'][:40],[]).append(float(x['Metric Value'])/1000)
    with open(f'gpurun_out/tr_kernels_{v}.txt','w') as f:
        for k,vv in d.items(): f.write(f"{k:40s} n={len(vv):3d} mean={sum(vv)/len(vv):8.2f} us\n")
PY
