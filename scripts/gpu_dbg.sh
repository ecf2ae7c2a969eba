mkdir -p gpurun_out
for D in 0 7 15 47 31 63 1 9; do
  echo "dbg=$D" >> gpurun_out/dbg.log
  HMC_TC_DBG=$D timeout 60 python scripts/tc_timeline.py 2>&1 | head -1 >> gpurun_out/dbg.log
  HMC_TC_DBG=$D HMC_TC_PRESPLIT=1 timeout 60 python scripts/tc_timeline.py 2>&1 | head -1 >> gpurun_out/dbg.log
done
