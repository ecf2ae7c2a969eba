#!/bin/bash
# A/B of the dT K split (dev build: HMC_DT_KS=1 disables it) on cfg4
mkdir -p gpurun_out/ab
for s in ${KS:-0 1 0 1}; do
  if [ $s = 0 ]; then unset HMC_DT_KS; else export HMC_DT_KS=$s; fi
  HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg cfg4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/cfg4.dtks$s.json 2>/dev/null
  echo "cfg4 dt_ks=$s (0 = planned split) $(python -c "import json;d=json.load(open('gpurun_out/ab/cfg4.dtks$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4), d['config']['engine'], d['acceptance'])" 2>&1)"
done
