"""Round-2 profile summaries -> profiles/: launch lists (share per kernel, cold-cache serialised),
the key metrics of the ncu --set full captures, and the bench lines of every config.
Reads gpurun_out/r2/ (scripts/r2_measure.sh, scripts/r2_ncu_full.sh)."""
import collections
import csv
import json
import os
import subprocess
import sys

R = os.environ.get("R2_DIR", "gpurun_out/r2")
OUT = os.environ.get("R2_OUT", "profiles")
UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def launches(cfg):
    rows = list(csv.reader(open(f"{R}/launches_{cfg}.csv")))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    H = rows[hdr]
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) != len(H):
            continue
        d = dict(zip(H, r))
        if d["Metric Name"] != "gpu__time_duration.sum":
            continue
        us = float(d["Metric Value"]) * UNIT.get(d["Metric Unit"], 1.0)
        name = d["Kernel Name"].split("(")[0]
        a = per.setdefault(name, [0.0, 0])
        a[0] += us
        a[1] += 1
    tot = sum(a[0] for a in per.values())
    out = [f"# ncu launch list, {cfg}: `python bench.py --cfg {cfg} --steps 1 --warmup 3 --L 2 --eps 4e-7 "
           f"--no-e2e --no-cpu-baseline` (first 400 launches; gpu__time_duration.sum, --clock-control none;",
           "# cold-cache and serialised: compare shares, not absolutes)", "  total us launches  share  kernel"]
    for name, (us, n) in sorted(per.items(), key=lambda kv: -kv[1][0]):
        out.append(f"{us:10.1f} {n:8d} {100 * us / tot:5.1f}%  {name}")
    return out


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__cluster_size",
        "smsp__inst_executed.sum", "sm__cycles_active.avg", "dram__bytes_read.sum.per_second",
        "dram__bytes_write.sum.per_second"]


def full(rep, title):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    out = [f"# ncu --set full --clock-control none: {title} ({os.path.basename(rep)})"]
    if len(rr) < 3:
        return out + ["  (no data)"]
    h, u = rr[0], rr[1]
    for v in rr[2:3]:
        d = {a: (b, c) for a, b, c in zip(h, v, u)}
        out.append("  kernel = " + d.get("Kernel Name", ("?", ""))[0][:160])
        for w in WANT:
            if w in d:
                out.append(f"  {w} = {d[w][0]} {d[w][1]}".rstrip())
    return out


def bench_lines():
    out = ["# bench lines (python bench.py --cfg <cfg> --steps 10|20 --warmup 3 --breakdown; one B200; "
           "scripts/r2_measure.sh)"]
    for c in ["cfg1", "cfg2", "cfg3", "cfg4", "cfg4u", "cfg5"]:
        p = f"{R}/final_{c}.json"
        if not os.path.exists(p):
            continue
        d = json.loads(open(p).read().strip().splitlines()[-1])
        json.dump(d, open(f"{OUT}/r02_bench_{c}.json", "w"), indent=1)
        r, w, cb, e = d["roofline"], d.get("whole_eval") or {}, d.get("cpu_baseline") or {}, d.get("e2e") or {}
        out.append(f"{c}: {d['value']:.0f} evals/s (e2e {e.get('value', 0):.0f}), {d['samples_per_s']:.1f} samples/s, "
                   f"{d['ms_per_step']:.2f} ms/step, acceptance {d['acceptance']:.3f}; dominant {r['kernel']} "
                   f"{r['achieved']:.1f} {r['unit']} = {r['frac']:.3f} of {r['peak']:.1f} ({r['bound']}); whole "
                   f"evaluation {w.get('frac', float('nan')):.3f}; oracle {cb.get('value', 0):.3g} evals/s on "
                   f"{cb.get('cores')} cores; SM {d['clocks']['sm_mhz']} MHz {d['clocks']['reasons']}; "
                   f"engine {d['config']['engine']}")
    p = f"{R}/final_reference.json"
    if os.path.exists(p):
        d = json.loads(open(p).read().strip().splitlines()[-1])
        json.dump(d, open(f"{OUT}/r02_bench_reference_arm.json", "w"), indent=1)
        out.append(f"reference arm (fp64 oracle, cfg5): {d['value']:.2f} evals/s, {d['cpu_baseline']['cores']} cores")
    return out


if __name__ == "__main__":
    lines = bench_lines() + [""]
    for c in ["cfg5", "cfg4", "cfg2"]:
        if os.path.exists(f"{R}/launches_{c}.csv"):
            lines += launches(c) + [""]
    for rep, title in [(f"{R}/full_cfg5_wgrad.ncu-rep", "cfg5 weight-gradient GEMM (EPI_WGRAD), 64 chains"),
                       (f"{R}/full_cfg5_fwd.ncu-rep", "cfg5 forward GEMM (EPI_FWD, pre-split weights), 64 chains"),
                       (f"{R}/full_cfg2_narrow.ncu-rep", "cfg2 narrow-engine kernel (one launch = all L = 50 steps)"),
                       (f"{R}/full_cfg1_narrow.ncu-rep", "cfg1 narrow-engine kernel (one launch = all L = 20 steps)")]:
        if os.path.exists(rep):
            lines += full(rep, title) + [""]
    open(f"{OUT}/r02_ncu_summary.txt", "w").write("\n".join(lines) + "\n")
    print("\n".join(lines))
