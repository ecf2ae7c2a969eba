"""Aggregate an ncu --metrics dram__bytes_*,gpu__time_duration csv (tcgen05 GEMM launches of one
cfg5 gradient evaluation) into per-class DRAM traffic per evaluation -> profiles/ncu_traffic.json."""
import collections, csv, json, re, sys

src = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/traffic.csv"
rows = list(csv.reader(open(src)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "nsecond": 1e-9}
CLASS = {"0, 0, 1, 1": "tc_fwd", "1, 1, 0, 3": "tc_wgrad", "0, 0, 0, 4": "tc_combine", "0, 1, 1, 2": "tc_dgrad",
         "0, 1, 0, 2": "tc_dB", "1, 1, 0, 2": "tc_dT"}
per = collections.OrderedDict()
for d in data:
    per.setdefault(d["ID"], {"name": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"]) * SCALE[d["Metric Unit"]]
agg = collections.defaultdict(lambda: {"launches": 0, "dram_bytes": 0.0, "seconds": 0.0})
for m in per.values():
    t = re.search(r"<128, ([^>]*)>", m["name"])
    c = CLASS.get(t.group(1) if t else "", "other")
    a = agg[c]
    a["launches"] += 1
    a["dram_bytes"] += m["dram__bytes_read.sum"] + m["dram__bytes_write.sum"]
    a["seconds"] += m["gpu__time_duration.sum"]
# the capture covers whole evaluations: 40 tc launches = ... classes per eval from the launch counts
res = {}
for c, a in agg.items():
    res[c] = a
    print(f"{c:12s} {a['launches']:3d} launches {a['dram_bytes'] / 1e6:9.1f} MB {a['seconds'] * 1e6:9.1f} us")
json.dump(res, open("/tmp/traffic_agg.json", "w"), indent=1)
