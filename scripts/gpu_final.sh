mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 2>&1 | grep -v Warning | tail -5 > gpurun_out/gpu_tests_full.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --cfg cfg4u --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4u.json 2> gpurun_out/bench_cfg4u.err
