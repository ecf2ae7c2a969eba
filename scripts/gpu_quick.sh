# quick GPU check: engine tests, diag, bench breakdown; optional full tests (FULL=1)
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -15 > gpurun_out/engine.log
timeout 600 python scripts/diag_engines.py ${DIAG_CFGS:-cfg3 cfg5} 2>&1 | grep -v "^    " > gpurun_out/diag.log
timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench.log 2>&1
if [ -n "$FULL" ]; then timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -v Warning | tail -30 > gpurun_out/gpu_tests.log; fi
echo done
