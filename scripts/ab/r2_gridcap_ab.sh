#!/bin/bash
# A/B of capped tcgen05 grids (several tiles per CTA pair; dev build: HMC_TC_GRIDCAP pairs, HMC_TC_GRIDCAP_EPI
# bit mask over EPI ids: 1 STORE (dT slabs), 2 FWD, 4 DACT, 8 WGRAD, 16 RESID) on cfg4
mkdir -p gpurun_out/ab
run() {
  HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so timeout 400 python bench.py --cfg ${CFG:-cfg4} --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps > gpurun_out/ab/gc.json 2>/dev/null
  echo "${CFG:-cfg4} gridcap=${HMC_TC_GRIDCAP:-none} epi=${HMC_TC_GRIDCAP_EPI:-all} $(python -c "import json;d=json.load(open('gpurun_out/ab/gc.json'));print(round(d['value']), round(d['whole_eval']['eval_ms'],4))" 2>&1)"
}
run
for ce in ${SWEEP:-"16 4" "22 4" "32 4" "32 5" "32 20" "32 21" "16 5"}; do
  set -- $ce
  HMC_TC_GRIDCAP=$1 HMC_TC_GRIDCAP_EPI=$2 run
done
run
