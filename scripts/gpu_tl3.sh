mkdir -p gpurun_out
for V in 5 2 4; do HMC_TC_PROF=$V timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl3_v$V.log 2>&1; done
