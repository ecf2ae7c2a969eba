mkdir -p gpurun_out/mwg
ncu --set full --clock-control none --import-source on -k regex:k_wgrad_mask -s 4 -c 2 -o gpurun_out/mwg/mwg_cfg5 python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --eps-mode config --no-e2e --no-cpu-baseline > gpurun_out/mwg/ncu.log 2>&1; echo ncu_rc=$?
tail -3 gpurun_out/mwg/ncu.log
