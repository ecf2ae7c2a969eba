#!/bin/bash
# weight-gradient K split under the halved input-gradient grids: cap for all layers (HMC_KS_MAX) x cap of each net's last one (HMC_KS_LAST)
mkdir -p gpurun_out/ab
for ce in ${SWEEP:-"1 0" "2 0" "1 2" "1 4" "1 0" "2 0" "1 2" "1 4"}; do
  set -- $ce
  export HMC_KS_MAX=$1; if [ $2 = 0 ]; then unset HMC_KS_LAST; else export HMC_KS_LAST=$2; fi
  HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg ${CFG:-cfg4} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/ks2.json 2>/dev/null
  echo "${CFG:-cfg4} ks_max=$1 ks_last=$2 $(python -c "import json;d=json.load(open('gpurun_out/ab/ks2.json'));print(round(d['value']), round(d['whole_eval']['eval_ms'],4))" 2>&1)"
done
