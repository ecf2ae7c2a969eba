mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -1 > gpurun_out/pdl.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -1 >> gpurun_out/pdl.log
for P in 1 0; do
  echo "pdl=$P" >> gpurun_out/pdl.log
  HMC_TC_PDL=$P timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/pdl.log
done
