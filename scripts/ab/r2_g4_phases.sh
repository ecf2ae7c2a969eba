#!/bin/bash
for v in 0 1; do echo "G4=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_G4=$v python scripts/narrow_phases.py cfg2 | tail -10; done
