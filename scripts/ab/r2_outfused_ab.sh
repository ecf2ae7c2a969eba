#!/bin/bash
# MLP output layer in one pass (k_out_fused) vs out_fwd + colred + rank-1 kernels
mkdir -p gpurun_out/ab
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/ab/pytest_of.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/ab/pytest_of.log
for s in 0 1 0 1; do
  HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_OUT_FUSED=$s timeout 240 python bench.py --cfg cfg3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --breakdown > gpurun_out/ab/cfg3.of$s.json 2> gpurun_out/ab/cfg3.of$s.err
  echo "cfg3 out_fused=$s $(python -c "import json;d=json.load(open('gpurun_out/ab/cfg3.of$s.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1 | tail -1)"
  grep -E "out_|bias_grad|rank" gpurun_out/ab/cfg3.of$s.err
done
