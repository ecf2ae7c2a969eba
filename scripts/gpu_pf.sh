mkdir -p gpurun_out
for PF in 0 3 6 12; do
  echo "== pf $PF" >> gpurun_out/pf.log
  HMC_TC_PF=$PF timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc|^\{" | cut -c1-120 >> gpurun_out/pf.log
done
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2 >> gpurun_out/pf.log
echo done
