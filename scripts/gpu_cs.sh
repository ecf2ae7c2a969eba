mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sensitivity.py -q -x 2>&1 | tail -1 > gpurun_out/cs.log
for R in 1 2; do for T in 1 0; do
  echo "csreg=$T" >> gpurun_out/cs.log
  HMC_TC_CSREG=$T timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E '"value"|breakdown\] tc_dgrad' | cut -c1-80 >> gpurun_out/cs.log
done; done
