bash scripts/gpu_full.sh
for V in 2 4; do HMC_TC_PROF=$V timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl4_v$V.log 2>&1; done
