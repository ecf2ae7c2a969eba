set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python -m pytest tests/test_gpu_engine.py -q -rf 2>&1 | tail -40 > gpurun_out/engine.log
timeout 1500 python -m pytest tests -m gpu -q -rf --timeout 600 2>&1 | tail -60 > gpurun_out/gpu_tests.log
timeout 400 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_tc.log 2>&1
HMC_ENGINE=simt timeout 600 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_simt.log 2>&1
