mkdir -p gpurun_out
for CFG in cfg3 cfg4 cfg5; do
  timeout 60 python scripts/hang_check.py $CFG >> gpurun_out/hang.log 2>&1; echo "$CFG rc=$?" >> gpurun_out/hang.log
done
timeout 120 python scripts/tc_timeline.py > gpurun_out/tl.log 2>&1
timeout 900 bash scripts/gpu_roles.sh
