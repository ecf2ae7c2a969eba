mkdir -p gpurun_out
HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd.log 2>&1
HMC_TC_PROF=3 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_dgrad.log 2>&1
for D in 0 2 63 1; do
  echo "dbg=$D" >> gpurun_out/dbg_bench.log
  HMC_TC_DBG=$D timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc" >> gpurun_out/dbg_bench.log
done
