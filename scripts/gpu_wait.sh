mkdir -p gpurun_out
for L in libhmc_w0.so libhmc.so libhmc_w2.so; do
  for D in 0 63; do
    echo "$L dbg=$D" >> gpurun_out/wait.log
    HMC_LIB=$PWD/paper_2507_14652_b200/$L HMC_TC_DBG=$D timeout 60 python scripts/tc_timeline.py 2>&1 | head -1 >> gpurun_out/wait.log
  done
  HMC_LIB=$PWD/paper_2507_14652_b200/$L timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc|^\{" | cut -c1-120 >> gpurun_out/wait.log
done
