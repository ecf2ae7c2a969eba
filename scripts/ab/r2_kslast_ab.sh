#!/bin/bash
# A/B of the K split of the LAST weight-gradient GEMM of each net (the backward tail: nothing overlaps it) - dev build, HMC_KS_LAST
mkdir -p gpurun_out/ab
for c in ${CFGS:-cfg4}; do
  for s in ${KS:-0 4 0 4 3 8}; do
    if [ $s = 0 ]; then unset HMC_KS_LAST; else export HMC_KS_LAST=$s; fi
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/$c.kl$s.json 2>/dev/null
    echo "$c ks_last=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/$c.kl$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1)"
  done
done
