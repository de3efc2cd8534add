#!/bin/bash
# ncu --set full of the TransR step kernels named by $KRE (regex) on the fb15k_transr bench workload
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"${KRE:-k_tr_mv|k_tr_dm_tc}" -s 20 -c ${NK:-3} \
  -o gpurun_out/tr_full python bench.py --workload fb15k_transr --steps 10 --warmup 5 --no-cpu-baseline --e2e-steps 5 > gpurun_out/ncu_tr.log 2>&1
for k in $(echo "${KRE:-k_tr_mv|k_tr_dm_tc}" | tr '|' ' '); do
  ncu -i gpurun_out/tr_full.ncu-rep -k regex:$k --page details --csv > gpurun_out/tr_details_$k.csv 2>/dev/null
done
echo done
for k in $(echo "${KRE:-k_tr_mv|k_tr_dm_tc}" | tr '|' ' '); do
  ncu -i gpurun_out/tr_full.ncu-rep -k regex:$k --page source --csv --print-source sass > gpurun_out/tr_src_$k.csv 2>/dev/null
done
