#!/bin/bash
# bench lines of the configs a change touched (CFGS) + the cfg4 launch list; outputs under gpurun_out/r2/
mkdir -p gpurun_out/r2
O=gpurun_out/r2
for c in ${CFGS:-cfg3 cfg4}; do
  timeout 900 python bench.py --cfg $c --steps 10 --warmup 3 --breakdown > $O/final_$c.json 2> $O/final_$c.err; echo bench $c rc=$?
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_cfg4.csv \
  python bench.py --cfg cfg4 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_launch_cfg4.log 2>&1; echo launches cfg4 rc=$?
python scripts/kernel_timeline.py cfg4 > $O/tl_cfg4.txt 2>&1
