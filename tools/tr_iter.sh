# TransR iteration: tests (-k transr), bench line, launch list
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
if [ -z "$NOTEST" ]; then timeout 900 python -m pytest tests -q -m gpu -k "transr or rescal" -x -rfE > gpurun_out/pt.txt 2>&1; fi
python bench.py --workload fb15k_transr --steps 300 --warmup 20 --no-cpu-baseline --e2e-steps 50 > gpurun_out/b.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 200 -c 40 --csv --log-file gpurun_out/tr_launches.csv python bench.py --workload fb15k_transr --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 5 > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/tr_launches.csv')))
hdr=None; d=collections.OrderedDict()
for r in rows:
    if r and r[0]=='ID': hdr=r; continue
    if hdr and len(r)==len(hdr):
        x=dict(zip(hdr,r))
        d.setdefault(x['Kernel Name'][:40],[]).append(float(x['Metric Value'])/1000)
with open('gpurun_out/tr_kernels.txt','w') as f:
    for k,v in d.items(): f.write(f"{k:40s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us\n")
PY
