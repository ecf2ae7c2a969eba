mkdir -p gpurun_out
SHORT="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:${NCU_KERNEL:-ELi3EE} -s ${NCU_SKIP:-4} -c 1 -o gpurun_out/prof_top $SHORT > gpurun_out/ncu_top.log 2>&1
echo done
