#!/bin/bash
# Round-2 measurement pass (one GPU): bench lines for every config (CPU oracle beside them, e2e),
# the reference arm, ncu launch lists, per-class DRAM traffic of cfg5, and --set full captures of
# the top kernels.  Outputs under gpurun_out/r2/ (summaries are copied to profiles/ by hand).
set -u
mkdir -p gpurun_out/r2
O=gpurun_out/r2
for c in ${CFGS:-cfg1 cfg2 cfg3 cfg4 cfg4u cfg5}; do
  K=10; [ $c = cfg5 ] && K=20; [ $c = cfg3 ] && K=10
  timeout 900 python bench.py --cfg $c --steps $K --warmup 3 --breakdown > $O/final_$c.json 2> $O/final_$c.err; echo bench $c rc=$?
done
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/final_reference.json 2>&1; echo ref rc=$?
if [ -z "${NO_NCU:-}" ]; then
# launch lists (bench command shortened: 1 step of L = 2, fixed stable eps; cold-cache serialised)
for c in cfg2 cfg4 cfg5; do
  ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$c.csv \
    python bench.py --cfg $c --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_launch_$c.log 2>&1; echo launches $c rc=$?
done
# cfg5 per-class DRAM traffic: the tensor-core GEMM launches of one evaluation (27 after 2 evals of warm-up)
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:tc_gemm_kernel -s 54 -c 27 --csv --log-file $O/traffic_cfg5.csv \
  python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_traffic.log 2>&1; echo traffic rc=$?
# --set full: cfg5 weight-gradient GEMM (variant <128,1,1,0,3>) and forward GEMM, cfg2 narrow kernel
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'\(bool\)1, \(bool\)1, \(bool\)0, \(int\)3>'  -s 8 -c 1 \
  -o $O/full_cfg5_wgrad python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_full1.log 2>&1; echo full1 rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'\(bool\)0, \(bool\)0, \(bool\)1, \(int\)1>'  -s 8 -c 1 \
  -o $O/full_cfg5_fwd python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_full2.log 2>&1; echo full2 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 3 -c 1 \
  -o $O/full_cfg2_narrow python bench.py --cfg cfg2 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full3.log 2>&1; echo full3 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_narrow -s 3 -c 1 \
  -o $O/full_cfg1_narrow python bench.py --cfg cfg1 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > $O/ncu_full4.log 2>&1; echo full4 rc=$?
fi
ls -la $O | tail -40
# summaries on the box (the .ncu-rep files exceed gpurun's 64 MiB copy-back limit): profile text /
# bench lines under $O/prof, the per-class traffic csv kept, the reports deleted but the weight-gradient one
mkdir -p $O/prof
R2_DIR=$O R2_OUT=$O/prof python scripts/r2_profiles.py > $O/prof/summary.log 2>&1; echo summary rc=$?
python scripts/ncu_traffic.py $O/traffic_cfg5.csv > $O/prof/traffic.log 2>&1; cp /tmp/traffic_agg.json $O/prof/ 2>/dev/null
rm -f $O/full_cfg5_fwd.ncu-rep $O/full_cfg2_narrow.ncu-rep $O/full_cfg1_narrow.ncu-rep
du -sh gpurun_out
