mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "grad" 2>&1 | tail -1 > gpurun_out/wg.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc|\"value\"" | cut -c1-100 >> gpurun_out/wg.log
HMC_TC_PROF=5 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_wg.log 2>&1
