mkdir -p gpurun_out
timeout 200 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2 > gpurun_out/mn.log
timeout 600 python -m pytest tests/test_gpu_unaligned.py tests/test_gpu_parity.py -q -x -k "cfg4 or unaligned or tiny or deeponet or cfg5 or cfg3" 2>&1 | tail -2 >> gpurun_out/mn.log
timeout 300 python scripts/diag_engines.py cfg4 cfg5 2>&1 | grep " tc " >> gpurun_out/mn.log
timeout 600 python bench.py --cfg cfg4u --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown|\"value\"" | cut -c1-100 >> gpurun_out/mn.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e 2>&1 | grep -o '"value": [0-9.]*' >> gpurun_out/mn.log
