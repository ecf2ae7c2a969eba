mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sensitivity.py tests/test_gpu_unaligned.py -q -x 2>&1 | tail -1 > gpurun_out/bias.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown|\"value\"" | cut -c1-90 >> gpurun_out/bias.log
