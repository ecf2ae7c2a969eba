mkdir -p gpurun_out
for H in "20 20 20" "0 20 20" "0 0 20" "0 0 0"; do
  set -- $H
  echo "hint p=$1 c=$2 e=$3" >> gpurun_out/wait.log
  HMC_TC_HINT_P=$1 HMC_TC_HINT_C=$2 HMC_TC_HINT_E=$3 timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc_(fwd|wgrad|dgrad)|\"value\"" | cut -c1-90 >> gpurun_out/wait.log
done
