"""Summarise one kernel of an ncu --set full report into a small JSON
(the numbers DESIGN.md and bench.py's roofline.traffic cite).
usage: ncu_summary.py REPORT KERNEL_REGEX LABEL [ALGO_BYTES]"""
import csv
import json
import re
import subprocess
import sys

rep, kre, label = sys.argv[1], sys.argv[2], sys.argv[3]
algo = float(sys.argv[4]) if len(sys.argv) > 4 else None
if rep.endswith(".csv"):   # a `ncu -i REPORT --page raw --csv` export
    out = open(rep).read()
else:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
pick = None
for r in rows[2:]:
    d = dict(zip(h, r))
    if re.search(kre, d.get("Kernel Name", "")):
        pick = d
        break
if pick is None:
    sys.exit(f"no kernel matching {kre}")


def f(k):
    v = pick.get(k, "")
    try:
        return float(v.replace(",", ""))
    except ValueError:
        return None


rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
units = rows[1] if len(rows) > 1 else []
uh = dict(zip(h, units))
rd *= scale.get(uh.get("dram__bytes_read.sum", "byte"), 1)
wr *= scale.get(uh.get("dram__bytes_write.sum", "byte"), 1)
t_ms = f("gpu__time_duration.sum")
if uh.get("gpu__time_duration.sum") in ("usecond", "us"):
    t_ms /= 1e3
elif uh.get("gpu__time_duration.sum") in ("nsecond", "ns"):
    t_ms /= 1e6
stalls = {k.replace("smsp__average_warps_issue_stalled_", "").replace(
    "_per_issue_active.ratio", ""): f(k) for k in h
    if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")}
top = dict(sorted(((k, v) for k, v in stalls.items() if v), key=lambda x: -x[1])[:5])
res = {
    "kernel": pick.get("Kernel Name", "")[:120],
    "label": label,
    "source": f"ncu --set full --clock-control none ({rep})",
    "gpu__time_duration_ms": t_ms,
    "dram_bytes_read": rd,
    "dram_bytes_write": wr,
    "dram_bytes_per_launch": rd + wr,
    "algorithmic_bytes_per_launch": algo,
    "tensor_dmma_active_pct": f("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_active_pct": f("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": f("launch__registers_per_thread"),
    "achieved_occupancy_pct": f("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "top_stalls_per_issue": top,
}
print(json.dumps(res, indent=1))
