#!/bin/bash
mkdir -p gpurun_out/r2
python scripts/narrow_probe.py cfg2 5 > gpurun_out/r2/probe.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_narrow -c 2 -o gpurun_out/r2/narrow_cfg2 python scripts/narrow_probe.py cfg2 1 > gpurun_out/r2/ncu_narrow.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/r2/ncu_narrow.log; cat gpurun_out/r2/probe.log
