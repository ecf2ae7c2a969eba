mkdir -p gpurun_out
timeout 300 python scripts/diag_engines.py cfg3 cfg5 2>&1 | grep -v "^    " > gpurun_out/diag.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench_raw.log 2>&1
HMC_TC_PRESPLIT=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench_pre.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 2>&1 | tail -3 > gpurun_out/gpu_tests.log
