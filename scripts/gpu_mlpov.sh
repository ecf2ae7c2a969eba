mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sensitivity.py tests/test_gpu_adapt.py -q -x 2>&1 | tail -1 > gpurun_out/mlpov.log
for S in 2 1; do
  echo "streams=$S" >> gpurun_out/mlpov.log
  HMC_STREAMS=$S timeout 300 python bench.py --cfg cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/mlpov.log
  HMC_STREAMS=$S timeout 300 python bench.py --cfg cfg2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/mlpov.log
done
