#!/bin/bash
# per-launch tensor-pipe / issue / DRAM metrics of the cfg5 weight-gradient GEMMs (trunk: 2048 rows, branch: 512)
mkdir -p gpurun_out/r2
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__cycles_active.avg \
  --clock-control none -k regex:'tc_gemm_kernel' -s 40 -c 60 --csv --log-file gpurun_out/r2/tc_metrics_cfg5.csv \
  python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --eps-mode config --no-e2e --no-cpu-baseline > gpurun_out/r2/ncu_metrics.log 2>&1; echo rc=$?
