#!/bin/bash
# A/B of the branch / trunk backward stream assignment (dev build, HMC_SWAP_BT) on the DeepONet configs
mkdir -p gpurun_out/ab
for c in ${CFGS:-cfg5 cfg4}; do
  for s in ${SW:-1 0 1 0}; do
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_SWAP_BT=$s timeout 400 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/$c.sw$s.json 2>/dev/null
    echo "$c swap_bt=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/$c.sw$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1)"
  done
done
