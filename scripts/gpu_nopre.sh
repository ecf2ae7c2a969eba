mkdir -p gpurun_out
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench_pre.log 2>&1
HMC_TC_NOPRE=1 timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench_nopre.log 2>&1
HMC_TC_NOPRE=1 timeout 300 python scripts/diag_engines.py cfg5 2>&1 | grep -v "^    " > gpurun_out/diag_nopre.log
