mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sensitivity.py tests/test_gpu_edges.py -q -x 2>&1 | tail -1 > gpurun_out/narrow.log
timeout 300 python bench.py --cfg cfg3 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E '"value"|breakdown\] narrow' | cut -c1-80 >> gpurun_out/narrow.log
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E '"value"|breakdown\] narrow' | cut -c1-80 >> gpurun_out/narrow.log
