#!/bin/bash
# A/B of two builds on one box: the product library (new) against libhmc_dev.so (built before the change)
mkdir -p gpurun_out/ab
for c in ${CFGS:-cfg4 cfg5}; do
  for s in new old new old; do
    if [ $s = old ]; then export HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so; else unset HMC_LIB; fi
    timeout 400 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/lib_$c.$s.json 2>/dev/null
    echo "$c lib=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/lib_$c.$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1)"
  done
done
