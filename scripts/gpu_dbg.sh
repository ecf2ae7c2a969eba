mkdir -p gpurun_out
for D in 0 1 2 3 4 7; do
  for SH in "1 1 256 2048" "0 0 2048 256"; do
    set -- $SH
    echo "dbg=$D akm=$1 bkm=$2 K=$3 M=$4" >> gpurun_out/dbg.log
    HMC_TC_DBG=$D TL_AKM=$1 TL_BKM=$2 TL_K=$3 TL_M=$4 timeout 60 python scripts/tc_timeline.py 2>&1 | head -1 >> gpurun_out/dbg.log
  done
done
