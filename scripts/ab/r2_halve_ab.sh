#!/bin/bash
# A/B of the halved input-gradient grids (dev build: HMC_DACT_HALVE=0 disables) on cfg4
mkdir -p gpurun_out/ab
for s in ${HV:-1 0 1 0}; do
  HMC_DACT_HALVE=$s HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg ${CFG:-cfg4} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/hv$s.json 2>/dev/null
  echo "${CFG:-cfg4} dact_halve=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/hv$s.json'));print(round(d['value']), round(d['whole_eval']['eval_ms'],4), d['acceptance'])" 2>&1)"
done
