mkdir -p gpurun_out
for D in 0 2 1; do HMC_TC_DBG=$D HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl5_d$D.log 2>&1; done
