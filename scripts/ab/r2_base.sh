set -x
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -x -q > gpurun_out/r2/base_pytest.log 2>&1; echo pytest_rc=$?
for c in cfg1 cfg2 cfg3 cfg4 cfg5; do
  timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --breakdown > gpurun_out/r2/base_$c.json 2> gpurun_out/r2/base_$c.err; echo $c rc=$?
done
