#!/bin/bash
mkdir -p gpurun_out/ab
python -m pytest tests -m gpu -q -x > gpurun_out/ab/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ab/pytest.log
for c in ${CFGS:-cfg4 cfg5 cfg3}; do
  for s in 0 1 0 1; do
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_WS2=$s timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/$c.w$s.json 2>/dev/null
    echo "$c ws2=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/$c.w$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1)"
  done
done
python scripts/kernel_timeline.py cfg4 > gpurun_out/tl_cfg4.txt 2>&1
