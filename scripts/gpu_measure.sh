# Round measurement: bench JSON line (default args), ncu launch list of a short run of the same
# command, and one `ncu --set full` capture of the dominant kernel class (weight-gradient GEMM).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 900 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
SHORT="python bench.py --steps 1 --warmup 1 --L 2 --no-cpu-baseline --no-e2e --breakdown"
timeout 300 $SHORT > gpurun_out/short.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $SHORT > gpurun_out/ncu_list.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on --kernel-name-base mangled -k regex:${NCU_KERNEL:-ELi3EE} -s ${NCU_SKIP:-4} -c 1 -o gpurun_out/prof_top $SHORT > gpurun_out/ncu_top.log 2>&1
echo done
