mkdir -p gpurun_out/small
for k in k_fwd_narrow k_wgrad_narrow_p1; do
ncu --set full --clock-control none -k regex:"$k" -s 2 -c 2 -o "gpurun_out/small/$k" python bench.py --cfg cfg5 --steps 1 --warmup 3 --L 2 --eps 4e-7 --eps-mode config --no-e2e --no-cpu-baseline > gpurun_out/small/log.txt 2>&1; echo $k rc=$?
done
