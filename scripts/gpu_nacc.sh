mkdir -p gpurun_out
make -q 2>/dev/null; ls -la paper_2507_14652_b200/libhmc.so alt/
for L in paper_2507_14652_b200/libhmc.so alt/libhmc_nacc3.so; do
  echo "lib=$L" >> gpurun_out/nacc.log
  HMC_LIB=$PWD/$L timeout 120 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1 >> gpurun_out/nacc.log
  HMC_LIB=$PWD/$L timeout 60 python scripts/hang_check.py cfg5 >> gpurun_out/nacc.log 2>&1; echo "rc=$?" >> gpurun_out/nacc.log
  HMC_LIB=$PWD/$L timeout 300 python scripts/diag_engines.py cfg5 2>&1 | grep -v "^    " | grep " tc " >> gpurun_out/nacc.log
  HMC_LIB=$PWD/$L timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc|\"value\"" | cut -c1-120 >> gpurun_out/nacc.log
done
HMC_TC_PROF=5 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_wgrad.log 2>&1
HMC_LIB=$PWD/alt/libhmc_nacc3.so HMC_TC_PROF=5 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_wgrad3.log 2>&1
HMC_LIB=$PWD/alt/libhmc_nacc3.so HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd3.log 2>&1
