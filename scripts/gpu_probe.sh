mkdir -p gpurun_out
timeout 300 python scripts/probe_tc_rounding.py > gpurun_out/probe.log 2>&1
CMD="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_list.log 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 6 -c 3 -o gpurun_out/prof_tc $CMD > gpurun_out/ncu_full.log 2>&1
echo done
