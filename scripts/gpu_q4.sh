mkdir -p gpurun_out
timeout 120 python -m pytest tests/test_gpu_engine.py -q -x 2>&1 | tail -2 > gpurun_out/engine.log
for CFG in "cfg3 2" "cfg5 2" "cfg5 64" "cfg4 16"; do timeout 60 python scripts/hang_check.py $CFG >> gpurun_out/hang.log 2>&1; echo "$CFG rc=$?" >> gpurun_out/hang.log; done
timeout 300 python scripts/diag_engines.py cfg3 cfg4 cfg5 2>&1 | grep -v "^    " > gpurun_out/diag.log
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --breakdown > gpurun_out/bench.log 2>&1
echo "bench rc=$?" >> gpurun_out/bench.log
HMC_TC_PROF=2 timeout 120 python scripts/tc_timeline_hmc.py > gpurun_out/tl_fwd.log 2>&1
