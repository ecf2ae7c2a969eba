#!/bin/bash
mkdir -p gpurun_out/nsrc
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 3 -c 1 -o gpurun_out/nsrc/narrow_cfg2 \
  python bench.py --cfg cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/nsrc/log.txt 2>&1; echo rc=$?
ls -la gpurun_out/nsrc
