# Round measurement: bench JSON line (default args), ncu launch list of a short run of the same
# command, one `ncu --set full` capture of the dominant kernel class (weight-gradient GEMM), and
# per-launch DRAM traffic of every tensor-core GEMM of one evaluation.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
SHORT="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e --breakdown"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_list.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:tc_gemm -c 27 --csv --log-file gpurun_out/traffic.csv $SHORT > gpurun_out/ncu_traffic.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:${NCU_KERNEL:-ELi3EE} -s ${NCU_SKIP:-4} -c 1 -o gpurun_out/prof_top $SHORT > gpurun_out/ncu_top.log 2>&1
echo done
