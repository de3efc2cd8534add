"""Summarise an ncu report into profiles/ncu_traffic.json: per kernel, DRAM bytes per launch (dram__bytes_read.sum +
dram__bytes_write.sum), duration, tensor-pipe and DRAM throughput, averaged over the captured launches.

    python tools/ncu_traffic.py gpurun_out/prof.ncu-rep profiles/ncu_traffic.json "<how it was captured>"
"""
import csv, io, json, subprocess, sys

rep, out = sys.argv[1], sys.argv[2]
how = sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units, body = rows[0], rows[1], rows[2:]


def col(name):
    return hdr.index(name) if name in hdr else None


def val(r, name, scale_to=None):
    i = col(name)
    if i is None or not r[i]:
        return None
    v = float(r[i].replace(",", ""))
    u = units[i]
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}
    return v * mult.get(u, 1.0)


acc = {}
for r in body:
    name = r[col("Kernel Name")].split("(")[0].split("<")[0].replace("void ", "").replace("kge::", "").strip()
    a = acc.setdefault(name, {"n": 0, "dram": 0.0, "us": 0.0, "tensor": 0.0, "dram_pct": 0.0})
    a["n"] += 1
    a["dram"] += (val(r, "dram__bytes_read.sum") or 0) + (val(r, "dram__bytes_write.sum") or 0)
    a["us"] += val(r, "gpu__time_duration.sum") or 0
    a["tensor"] += val(r, "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active") or 0
    a["dram_pct"] += val(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed") or 0
res = {"source": rep, "how": how, "kernels": {}}
for k, a in acc.items():
    n = a["n"]
    res["kernels"][k] = {"launches": n, "dram_bytes_per_launch": a["dram"] / n, "us_per_launch": a["us"] / n,
                         "tensor_pipe_pct_active": a["tensor"] / n, "dram_throughput_pct": a["dram_pct"] / n}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
