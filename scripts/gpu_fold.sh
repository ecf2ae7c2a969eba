mkdir -p gpurun_out
./scripts/micro/tmem_bw > gpurun_out/tmem_bw.log 2>&1
for F in 1 2 4; do
  echo "== fold $F" >> gpurun_out/fold.log
  HMC_TC_FOLD=$F timeout 600 python scripts/diag_engines.py cfg3 cfg5 2>&1 | grep " tc " >> gpurun_out/fold.log
  HMC_TC_FOLD=$F timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown|^\{" | cut -c1-200 >> gpurun_out/fold.log
done
timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -v Warning | tail -5 > gpurun_out/gpu_tests.log
echo done
