mkdir -p gpurun_out
for D in 0 128; do HMC_TC_DBG=$D HMC_TC_PROF=4 HMC_STREAMS=1 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_dact_$D.log 2>&1; done
