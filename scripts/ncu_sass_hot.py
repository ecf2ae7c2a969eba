"""Dev: hottest SASS instructions of a kernel in an ncu report (warp-stall samples), with
shared-memory wavefront excess.  usage: ncu_sass_hot.py report.ncu-rep kernel_regex [launch#] [top]"""
import collections
import csv
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
nth = sys.argv[3] if len(sys.argv) > 3 else "1"
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "--kernel-id", f"::regex:{kre}:{nth}"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
ix = {n: i for i, n in enumerate(h)}
recs = []
for r in rows[2:]:
    if len(r) != len(h):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    recs.append((s, r[ix["Address"]], r[ix["Source"]].strip(), int(r[ix["Instructions Executed"]] or 0),
                 r[ix.get("L1 Wavefronts Shared Excessive", 0)], r[ix.get("L1 Wavefronts Shared", 0)]))
tot = sum(x[0] for x in recs)
ops = collections.Counter()
execd = collections.Counter()
for s, a, src, ex, _, _ in recs:
    op = src.split()[0] if src else "?"
    if op.startswith("@"):
        op = src.split()[1]
    ops[op.split(".")[0]] += s
    execd[op.split(".")[0]] += ex
print(f"total samples {tot}, instructions executed {sum(execd.values())}")
print("by opcode (samples %, executed):")
for op, s in ops.most_common(20):
    print(f"  {op:10s} {100 * s / max(tot, 1):5.1f}%  {execd[op]}")
print("hottest instructions:")
for s, a, src, ex, wx, w in sorted(recs, reverse=True)[:top]:
    print(f"  {100 * s / max(tot, 1):5.2f}% {a[-5:]} ex={ex:9d} shw={w}/{wx}x  {src[:90]}")
