mkdir -p gpurun_out
for R in 1 2; do for F in 1 0; do
  echo "fuse=$F" >> gpurun_out/ab.log
  HMC_BIAS_FUSE=$F timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/ab.log
done; done
