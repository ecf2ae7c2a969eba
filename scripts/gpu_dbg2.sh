mkdir -p gpurun_out
for D in 0 64 2 66 63; do
  echo "dbg=$D" >> gpurun_out/dbg2.log
  HMC_TC_DBG=$D timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc" >> gpurun_out/dbg2.log
done
