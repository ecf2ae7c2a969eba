#!/bin/bash
# K-split A/B of the weight-gradient GEMMs inside the concurrent backward (dev build, HMC_KS_MAX)
mkdir -p gpurun_out/ab
for c in ${CFGS:-cfg4 cfg3}; do
  for s in ${KS:-16 1 2 16 1 2}; do
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_KS_MAX=$s timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/$c.ks$s.json 2>/dev/null
    echo "$c ks_max=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/$c.ks$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1)"
  done
done
