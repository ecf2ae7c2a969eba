#!/bin/bash
mkdir -p gpurun_out/r2
timeout 600 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_parity.py -q -x -k "narrow or cfg1 or cfg2 or blr or deep_narrow or L0 or batch" > gpurun_out/r2/narrow_pytest.log 2>&1; echo pytest_rc=$?
tail -5 gpurun_out/r2/narrow_pytest.log
python scripts/narrow_probe.py cfg2 5; python scripts/narrow_probe.py cfg1 5
for c in cfg1 cfg2; do
  timeout 300 python bench.py --cfg $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --breakdown > gpurun_out/r2/narrow_$c.json 2> gpurun_out/r2/narrow_$c.err; echo $c rc=$?
  tail -3 gpurun_out/r2/narrow_$c.err
done
if [ -n "$NCU" ]; then
ncu --set full --clock-control none --import-source on -k regex:k_narrow -c 2 -o gpurun_out/r2/narrow_cfg2_v2 python scripts/narrow_probe.py cfg2 1 > gpurun_out/r2/ncu_narrow.log 2>&1; echo ncu_rc=$?
fi
