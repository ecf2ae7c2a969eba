#!/bin/bash
# masked weight gradient: GPU tests on the product build, then A/B (dense GEMM vs masked) per config
# on the developer build (HMC_MWG=0 / 1)
mkdir -p gpurun_out/mwg
python -m pytest tests -m gpu -x -q > gpurun_out/mwg/pytest.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/mwg/pytest.log
for c in ${CFGS:-cfg3 cfg4 cfg5}; do
  for m in 0 1; do
    HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_MWG=$m timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps --breakdown > gpurun_out/mwg/$c.$m.json 2> gpurun_out/mwg/$c.$m.err
    echo "$c mwg=$m rc=$? $(python -c "import json;d=json.load(open('gpurun_out/mwg/$c.$m.json'));print(round(d['value']), d['clocks']['sm_mhz'], d['config']['engine'])" 2>&1)"
    grep -E "wgrad|fwd|dgrad" gpurun_out/mwg/$c.$m.err | head -6
  done
done
