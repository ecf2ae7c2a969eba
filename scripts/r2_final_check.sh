#!/bin/bash
# what the driver runs at round end: GPU tests, smoke, the default bench line and the reference arm
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q -x > gpurun_out/r2/final_pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/r2/final_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/final_smoke.log 2>&1; echo smoke_rc=$?
python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2/final_ref_default.json 2>&1; echo ref_rc=$?
python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2/final_default.json 2> gpurun_out/r2/final_default.err; echo bench_rc=$?
tail -c 400 gpurun_out/r2/final_default.json
