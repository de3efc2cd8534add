"""Top SASS instructions by warp-stall samples from an ncu report (source page)."""
import csv, io, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name", f"regex:{kern}"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr, body = rows[0], rows[1:]
ia, isrc, iss = hdr.index("Address"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iss]) for r in body if r[iss].isdigit())
body = [(int(r[iss]), n, r[isrc].strip()) for n, r in enumerate(body) if r[iss].isdigit()]
print("total samples", tot)
for s, n, src in sorted(body, reverse=True)[:top]:
    print(f"{s:6d} {100*s/tot:5.1f}%  #{n:5d}  {src}")
if len(sys.argv) > 4:  # phase split: comma-separated instruction-index boundaries
    cuts = [int(x) for x in sys.argv[4].split(",")]
    acc = [0] * (len(cuts) + 1)
    for s, n, _ in body:
        k = sum(n >= c for c in cuts)
        acc[k] += s
    print("phases", cuts, [f"{100*a/tot:.1f}%" for a in acc])
