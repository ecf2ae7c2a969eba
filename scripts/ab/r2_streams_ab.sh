#!/bin/bash
# concurrency A/B: default (captured branch / trunk and weight-gradient streams) vs one stream
mkdir -p gpurun_out/ab
for c in ${CFGS:-cfg5 cfg3 cfg4}; do
  for s in 0 1 0 1; do
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_STREAMS=$s timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/$c.s$s.json 2>/dev/null
    echo "$c streams=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/$c.s$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4), round(d['whole_eval']['eval_ms_profiled_single_stream'],4))" 2>&1)"
  done
done
