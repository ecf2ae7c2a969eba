mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sensitivity.py -q -x 2>&1 | tail -1 > gpurun_out/q5.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/q5_bench.json 2> gpurun_out/q5_bench.err
grep -E "breakdown" gpurun_out/q5_bench.err >> gpurun_out/q5.log
