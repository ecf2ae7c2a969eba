mkdir -p gpurun_out
timeout 600 python scripts/cost_compare.py cfg4 150 > gpurun_out/cost_cfg4.json 2> gpurun_out/cost_cfg4.err
timeout 600 python scripts/cost_compare.py cfg2 200 > gpurun_out/cost_cfg2.json 2> gpurun_out/cost_cfg2.err
bash scripts/gpu_measure.sh
