mkdir -p gpurun_out
for R in 1 2; do for T in 1 0; do
  echo "tanh_end=$T" >> gpurun_out/te2.log
  HMC_TC_TANHEND=$T timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/te2.log
done; done
