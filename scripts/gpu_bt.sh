mkdir -p gpurun_out
for B in 0 1; do
  echo "btrunc=$B" >> gpurun_out/bt.log
  HMC_TC_BTRUNC=$B timeout 300 python scripts/diag_engines.py cfg3 cfg5 2>&1 | grep -v "^    " | grep " tc " >> gpurun_out/bt.log
  HMC_TC_BTRUNC=$B timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc_wgrad" >> gpurun_out/bt.log
done
