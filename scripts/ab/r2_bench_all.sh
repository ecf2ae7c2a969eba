#!/bin/bash
# one bench line per config (round 2): gpurun_out/r2/bench_<cfg>.json
mkdir -p gpurun_out/r2
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg4 cfg5}; do
  timeout 600 python bench.py --cfg $c --steps ${K:-10} --warmup ${W:-3} --breakdown ${EXTRA:-} > gpurun_out/r2/bench_$c.json 2> gpurun_out/r2/bench_$c.err; echo $c rc=$?
  tail -4 gpurun_out/r2/bench_$c.err
done
