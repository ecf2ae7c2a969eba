#!/bin/bash
# round-end style check: GPU tests, smoke, default bench line, reference arm, torchrun DATA mode at N = 1,
# and the ncu --set full capture of a cfg5 TRUNK weight-gradient launch (the longest of 4)
bash scripts/r2_final_check.sh
mkdir -p gpurun_out/r2
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 2 --warmup 3 --cfg cfg5 --parallel data > gpurun_out/r2/torchrun_data.json 2> gpurun_out/r2/torchrun_data.err; echo torchrun_rc=$?
tail -c 300 gpurun_out/r2/torchrun_data.json
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'\(bool\)1, \(bool\)1, \(bool\)0, \(int\)3>' -s 8 -c 4 \
  -o gpurun_out/r2/full_cfg5_wgrad4 python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --eps-mode config --no-e2e --no-cpu-baseline > gpurun_out/r2/ncu_full5.log 2>&1; echo full5 rc=$?
python - <<'PY'
import csv, subprocess
raw = subprocess.run(["ncu", "-i", "gpurun_out/r2/full_cfg5_wgrad4.ncu-rep", "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "sm__cycles_active.avg"]
with open("gpurun_out/r2/full_cfg5_wgrad4.txt", "w") as f:
    for v in rr[2:]:
        d = dict(zip(h, v))
        f.write("launch " + d.get("ID", "?") + ": " + "; ".join(f"{k} = {d.get(k)} {dict(zip(h, rr[1])).get(k, '')}" for k in keys) + "\n")
print(open("gpurun_out/r2/full_cfg5_wgrad4.txt").read())
PY
rm -f gpurun_out/r2/full_cfg5_wgrad4.ncu-rep
