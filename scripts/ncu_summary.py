"""Build profiles/r01_ncu_summary.txt from the artifacts of scripts/gpu_measure.sh: the ncu launch
list (gpurun_out/launches.csv), the per-class DRAM traffic (profiles/ncu_traffic.json) and the
`ncu --set full` capture of the top kernel (gpurun_out/prof_top.ncu-rep, read with `ncu -i`)."""
import collections
import csv
import json
import subprocess
import sys

OUT = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_ncu_summary.txt"
lines = []

# ---- launch list ----
rows = list(csv.reader(open("gpurun_out/launches.csv")))
hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
H = rows[hdr]
per = collections.OrderedDict()
for r in rows[hdr + 1:]:
    if len(r) != len(H):
        continue
    d = dict(zip(H, r))
    if d["Metric Name"] != "gpu__time_duration.sum":
        continue
    v = float(d["Metric Value"]) * {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3, "ns": 1e-3, "us": 1.0}.get(d["Metric Unit"], 1.0)
    name = d["Kernel Name"]
    name = name.split("(")[0] if "(" in name else name
    a = per.setdefault(name, [0.0, 0])
    a[0] += v
    a[1] += 1
tot = sum(a[0] for a in per.values())
lines.append("# ncu launch list, `python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e --breakdown`")
lines.append("# (gpu__time_duration.sum, --clock-control none; cold-cache serialised: compare shares)")
lines.append("  total us launches  share  kernel")
for name, (us, n) in sorted(per.items(), key=lambda kv: -kv[1][0]):
    lines.append(f"{us:10.1f} {n:8d} {100 * us / tot:5.1f}%  {name}")

# ---- traffic ----
tr = json.load(open("profiles/ncu_traffic.json"))
lines.append("")
lines.append("# DRAM traffic per gradient evaluation (64 chains) by tensor-core GEMM class (profiles/ncu_traffic.json)")
for c, b in tr["cfg5"].items():
    n = tr.get("_per_class_launches", {}).get(c, 0)
    s = tr.get("_per_class_seconds_serialised", {}).get(c, 0.0)
    lines.append(f"{c:12s} {n:3d} launches {b / 1e6:9.1f} MB {s * 1e6:9.1f} us")

# ---- top kernel, ncu --set full ----
raw = subprocess.run(["ncu", "-i", "gpurun_out/prof_top.ncu-rep", "--page", "raw", "--csv"],
                     capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
if len(rr) >= 3:
    h, u, v = rr[0], rr[1], rr[2]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
            "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_size",
            "smsp__inst_executed.sum"]
    lines.append("")
    lines.append("# ncu --set full, top kernel class (" + sys.argv[2] if len(sys.argv) > 2 else "# ncu --set full, top kernel class")
    for w in want:
        if w in h:
            i = h.index(w)
            lines.append(f"  {w} = {v[i]} {u[i]}".rstrip())
open(OUT, "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
