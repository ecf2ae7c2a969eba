#!/bin/bash
# GPU tests + short bench lines of the named configs (breakdown to stderr)
mkdir -p gpurun_out/q
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/q/pytest.log 2>&1; echo pytest_rc=$?; tail -2 gpurun_out/q/pytest.log
for c in ${CFGS:-cfg3 cfg5}; do
  timeout 300 python bench.py --cfg $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-config-eps --breakdown > gpurun_out/q/$c.json 2> gpurun_out/q/$c.err
  echo "$c $(python -c "import json;d=json.load(open('gpurun_out/q/$c.json'));print(round(d['value']), d['clocks']['sm_mhz'], round(d['whole_eval']['eval_ms'],4))" 2>&1 | tail -1)"
  grep -E "narrow|out_f" gpurun_out/q/$c.err
done
