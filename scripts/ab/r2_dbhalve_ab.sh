#!/bin/bash
# A/B: dB (head of the branch backward chain) with its full grid vs the halved one (dev build, HMC_DB_HALVE=0)
mkdir -p gpurun_out/ab
for s in ${HV:-1 0 1 0}; do
  HMC_DB_HALVE=$s HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg ${CFG:-cfg4} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/dbh$s.json 2>/dev/null
  echo "${CFG:-cfg4} db_halve=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/dbh$s.json'));print(round(d['value']), round(d['whole_eval']['eval_ms'],4))" 2>&1)"
done
