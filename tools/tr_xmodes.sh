#!/bin/bash
# TransR timing experiments by KGE_TR_XMODE (0 normal, 1 no projection epilogue stores, 2 no score pair loop,
# 3 no dQ stores) -- numbers are timings only (modes 1-3 compute wrong results)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
for m in 0 1 2 3; do
  KGE_TR_XMODE=$m ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_tr_tc|k_tr_score|k_tr_dm" -s 10 -c 10 --csv --log-file gpurun_out/x_$m.csv python bench.py --workload fb15k_transr --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 5 > /dev/null 2>&1
done
python - <<'PY'
import csv, collections
for m in range(4):
    rows=list(csv.reader(open(f'gpurun_out/x_{m}.csv')))
    hdr=None; d=collections.OrderedDict()
    for r in rows:
        if r and r[0]=='ID': hdr=r; continue
        if hdr and len(r)==len(hdr):
            x=dict(zip(hdr,r)); d.setdefault(x['Kernel Name'][:22],[]).append(float(x['Metric Value'])/1000)
    print(m, {k: round(sum(v)/len(v),1) for k,v in d.items()})
PY
