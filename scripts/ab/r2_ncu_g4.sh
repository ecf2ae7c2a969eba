#!/bin/bash
mkdir -p gpurun_out/g4
for v in 1 0; do
HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_G4=$v timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 1 -c 1 -o gpurun_out/g4/narrow_g4_$v \
  python scripts/narrow_probe.py cfg2 2 > gpurun_out/g4/log_$v.txt 2>&1; echo rc=$?
done
ls -la gpurun_out/g4
