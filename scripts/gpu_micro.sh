mkdir -p gpurun_out
./scripts/micro/mma_rate > gpurun_out/mma_rate.log 2>&1
SHORT="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:tc_gemm -c 40 --csv --log-file gpurun_out/traffic.csv $SHORT > gpurun_out/ncu_traffic.log 2>&1
echo done
