# dev loop on the GPU box: engine + diag + parity tests + bench
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -15 > gpurun_out/engine.log
timeout 600 python scripts/diag_engines.py ${DIAG_CFGS:-cfg3 cfg5} > gpurun_out/diag.log 2>&1
if [ -z "$SKIP_TESTS" ]; then timeout 1200 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -v Warning | tail -40 > gpurun_out/gpu_tests.log; fi
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --breakdown > gpurun_out/bench.log 2>&1
echo done
