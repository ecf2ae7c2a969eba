#!/bin/bash
for v in 0 1 0 1; do echo "G4=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_G4=$v python scripts/narrow_probe.py cfg2 20 | tail -1; done
bash scripts/ab/r2_g4_phases.sh
