mkdir -p gpurun_out
timeout 300 python scripts/diag_engines.py cfg5 2>&1 | grep " tc " > gpurun_out/te.log
for T in 1 0; do
  echo "tanh_end=$T" >> gpurun_out/te.log
  HMC_TC_TANHEND=$T timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc_fwd|\"value\"" | cut -c1-100 >> gpurun_out/te.log
done
HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd.log 2>&1
