mkdir -p gpurun_out/r2
ncu --set full --clock-control none -k regex:k_leapfrog -s 3 -c 1 -o gpurun_out/r2/full_leapfrog python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --no-e2e --no-cpu-baseline > gpurun_out/r2/ncu_lf.log 2>&1; echo rc=$?
timeout 600 python scripts/project_scaling.py cfg5 3 points_xc > /dev/null 2>&1; echo proj=$?
