mkdir -p gpurun_out/r2
for lib in ./alt_f4.so; do
  echo "== $lib"
  HMC_LIB=$lib python bench.py --cfg cfg5 --steps 5 --warmup 3 --eps 4e-7 --no-e2e --no-cpu-baseline --breakdown > gpurun_out/r2/f4_$(basename $lib).json 2> gpurun_out/r2/f4_$(basename $lib).err
  python -c "
import json; d=json.loads(open('gpurun_out/r2/f4_$(basename $lib).json').read().strip().splitlines()[-1]); print(round(d['value']), d['ms_per_step'], d['clocks']['sm_mhz'], d['whole_eval']['frac'])"
  head -7 gpurun_out/r2/f4_$(basename $lib).err
done
HMC_LIB=./alt_f4.so python -m pytest tests/test_gpu_parity.py -q -x -k "full_configs or engines_agree or tiny or resynced_20 or every_20th" 2>&1 | tail -3
HMC_LIB=./alt_f4.so python scripts/diag_engines.py cfg3 cfg5 2>&1 | grep -v "    " | head -10
