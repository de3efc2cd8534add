"""Markdown tables from a gpurun evidence run (tools/gpu_full.sh): bench line, per-config lines, launch list, ncu
capture. Used to write profiles/r01_summary.md.

    python tools/summarize_round.py gpurun_out
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

d = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out"


def jline(path):
    if not os.path.exists(path):
        return None
    ls = [x for x in open(path) if x.startswith("{")]
    return json.loads(ls[-1]) if ls else None


b = jline(os.path.join(d, "bench.log"))
if b:
    r = b["roofline"]
    print(f"bench: {b['value'] / 1e6:.2f} M pos/s, {b['ms_per_step'] * 1e3:.2f} us/step, e2e {b['e2e']['value'] / 1e6:.2f} M, "
          f"launches {b['gpu_launches']}, clocks {b['clocks']}, cpu {b['cpu_baseline']}")
    print(f"roofline dominant {r['kernel']} {r['bound']} {r['achieved']:.1f} {r['unit']} frac {r['frac']:.4f} "
          f"traffic {r['traffic']} share {r['share_of_step']:.3f}; step_hbm {r['step_hbm']}")
    print("| kernel | isolated us | bound | achieved | frac | ncu DRAM bytes |")
    print("|---|---|---|---|---|---|")
    for k, v in r["kernels"].items():
        print(f"| {k} | {v['ms'] * 1e3:.2f} | {v['bound']} | {v['achieved']:.1f} {v['unit']} | {v['frac']:.4f} | {v['traffic']} |")
ref = jline(os.path.join(d, "bench_ref.log"))
if ref:
    print(f"reference arm: {ref.get('value')} {ref.get('unit')} ({ref.get('cpu_baseline', {}).get('sample')})")
cfg = os.path.join(d, "configs.log")
if os.path.exists(cfg):
    print("\n| config | M pos/s | us/step | e2e M pos/s | dominant kernel (isolated) | bound | frac | per-kernel isolated us | CPU oracle pos/s |")
    print("|---|---|---|---|---|---|---|---|---|")
    cur = None
    for line in open(cfg):
        if line.startswith("=="):
            cur = line[3:].strip()
            continue
        if line.startswith("{"):
            x = json.loads(line)
            r = x["roofline"]
            per = ", ".join(f"{k.replace('k_', '')} {v * 1e3:.1f}" for k, v in r["per_kernel_ms"].items() if v)
            cb = x.get("cpu_baseline") or {}
            print(f"| `{cur}` | {x['value'] / 1e6:.2f} | {x['ms_per_step'] * 1e3:.1f} | {x['e2e']['value'] / 1e6:.2f} | "
                  f"{r['kernel']} | {r['bound']} | {(r['frac'] or 0):.4f} | {per} | {cb.get('value', 0):.0f} |")
lc = os.path.join(d, "launches.csv")
if os.path.exists(lc):
    rows = list(csv.reader(open(lc)))
    i = [n for n, rr in enumerate(rows) if rr and rr[0] == "ID"][0]
    hdr, body = rows[i], rows[i + 1:]
    kn, mv = hdr.index("Kernel Name"), hdr.index("Metric Value")
    acc = collections.defaultdict(list)
    for rr in body:
        acc[rr[kn].split("(")[0].split("<")[0].replace("void ", "").replace("kge::", "")].append(float(rr[mv].replace(",", "")))
    tot = sum(sum(v) for v in acc.values())
    print("\n| kernel (ncu launch list) | launches | avg us | share |")
    print("|---|---|---|---|")
    for k, v in sorted(acc.items(), key=lambda kv: -sum(kv[1])):
        print(f"| {k} | {len(v)} | {sum(v) / len(v) / 1000:.2f} | {sum(v) / tot:.3f} |")
