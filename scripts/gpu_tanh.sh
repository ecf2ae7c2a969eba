mkdir -p gpurun_out
timeout 60 ./scripts/micro/tanh_rate > gpurun_out/tanh_rate.log 2>&1
HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd.log 2>&1
HMC_TC_DBG=64 HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd64.log 2>&1
for D in 0 64; do
  echo "dbg=$D" >> gpurun_out/dbg_tanh.log
  HMC_TC_DBG=$D timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc" >> gpurun_out/dbg_tanh.log
done
