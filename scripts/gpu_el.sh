mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_datamode.py -q -x 2>&1 | tail -1 > gpurun_out/el.log
for R in 1 2; do for E in 1 0; do
  echo "emit_lead=$E" >> gpurun_out/el.log
  HMC_TC_EMITLEAD=$E timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E '"value"|breakdown\] tc_(combine|dgrad|dB|dT)' | cut -c1-80 >> gpurun_out/el.log
done; done
