mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grad" 2>&1 | tail -1 > gpurun_out/rawb.log
HMC_TC_RAWB=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grad" 2>&1 | tail -1 >> gpurun_out/rawb.log
for R in 1 2; do for B in 1 0; do
  echo "rawb=$B" >> gpurun_out/rawb.log
  HMC_TC_RAWB=$B timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/rawb.log
done; done
