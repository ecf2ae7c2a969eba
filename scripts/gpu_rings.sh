mkdir -p gpurun_out
for L in paper_2507_14652_b200/libhmc.so alt/libhmc_s6468.so alt/libhmc_s5568.so; do
  echo "lib=$L" >> gpurun_out/rings.log
  HMC_LIB=$PWD/$L timeout 120 python scripts/hang_check.py cfg5 64 >> gpurun_out/rings.log 2>&1
  HMC_LIB=$PWD/$L timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc|\"value\"" | cut -c1-90 >> gpurun_out/rings.log
done
