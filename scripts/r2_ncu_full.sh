set -u
O=gpurun_out/r2
mkdir -p $O
# --set full: cfg5 weight-gradient GEMM (variant <128,1,1,0,3>) and forward GEMM, cfg2 narrow kernel
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'\(bool\)1, \(bool\)1, \(bool\)0, \(int\)3>'  -s 8 -c 1 \
  -o $O/full_cfg5_wgrad python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_full1.log 2>&1; echo full1 rc=$?
ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:'\(bool\)0, \(bool\)0, \(bool\)1, \(int\)1>'  -s 8 -c 1 \
  -o $O/full_cfg5_fwd python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > $O/ncu_full2.log 2>&1; echo full2 rc=$?
