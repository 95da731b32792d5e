"""Top source lines / SASS by warp-stall samples from an ncu report."""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = next(r for r in rows if "Warp Stall Sampling (All Samples)" in r)
si = hdr.index("Warp Stall Sampling (All Samples)")
start = rows.index(hdr) + 1
lines, sass = [], []
for r in rows[start:]:
    if len(r) <= si:
        continue
    try:
        v = int(r[si])
    except ValueError:
        continue
    if r[0] != "":
        lines.append((v, r[0], r[1][:100]))
    else:
        sass.append((v, r[3][:90] if len(r) > 3 else ""))
tot = max(sum(x[0] for x in lines), 1)
for v, ln, src in sorted(lines, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}%  line {ln}: {src}")
print("--- sass")
tot = max(sum(x[0] for x in sass), 1)
for v, s in sorted(sass, reverse=True)[:n]:
    print(f"{v / tot * 100:5.1f}%  {s}")
