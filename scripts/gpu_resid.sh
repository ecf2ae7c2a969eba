mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_datamode.py tests/test_gpu_edges.py -q -x 2>&1 | tail -1 > gpurun_out/resid.log
for R in 1 2; do
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E '"value"|breakdown\] tc_combine' | cut -c1-80 >> gpurun_out/resid.log
done
