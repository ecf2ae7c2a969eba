mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2 > gpurun_out/engine.log
timeout 300 python scripts/tc_roles.py > gpurun_out/roles.log 2>&1
timeout 600 python scripts/diag_engines.py cfg3 cfg4 cfg5 2>&1 | grep -v "^    " > gpurun_out/diag.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench.log 2>&1
echo done
if [ -n "$FULL" ]; then timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -v Warning | tail -5 > gpurun_out/gpu_tests.log; fi
