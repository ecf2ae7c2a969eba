mkdir -p gpurun_out
timeout 300 python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/pre_ncu.log 2>&1 && \
timeout 900 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:ILi128ELb0ELb0ELb1ELi1E --launch-skip 6 --launch-count 1 -o gpurun_out/prof_fwd -f python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e > gpurun_out/ncu_fwd.log 2>&1
echo rc=$? >> gpurun_out/ncu_fwd.log
