mkdir -p gpurun_out
for H in "20 20 20" "1000 20 20" "1000 200 20" "1000 1000 20" "1000 1000 200" "5000 5000 20" "100000 100000 100000"; do
  set -- $H
  echo "hint p=$1 c=$2 e=$3" >> gpurun_out/hint.log
  HMC_TC_HINT_P=$1 HMC_TC_HINT_C=$2 HMC_TC_HINT_E=$3 timeout 300 python bench.py --steps 1 --warmup 3 --L 20 --no-cpu-baseline --no-e2e --breakdown 2>&1 | grep -E "breakdown\] tc_(fwd|wgrad|dgrad)" >> gpurun_out/hint.log
done
