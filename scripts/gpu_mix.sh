mkdir -p gpurun_out
for L in paper_2507_14652_b200/libhmc.so alt/libhmc_mix.so; do
  echo "lib=$L" >> gpurun_out/mix.log
  HMC_LIB=$PWD/$L timeout 300 python scripts/diag_engines.py cfg5 2>&1 | grep " tc " >> gpurun_out/mix.log
  HMC_LIB=$PWD/$L timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc_fwd|\"value\"" | cut -c1-90 >> gpurun_out/mix.log
done
