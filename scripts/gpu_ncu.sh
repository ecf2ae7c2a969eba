# ncu capture of the tcgen05 GEMMs of one cfg5 eval (after a plain run of the same command)
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s ${NCU_SKIP:-4} -c ${NCU_COUNT:-8} -o gpurun_out/prof_tc2 $CMD > gpurun_out/ncu_full.log 2>&1
echo done
