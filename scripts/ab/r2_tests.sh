#!/bin/bash
# GPU test pass + smoke (round 2 iterations)
mkdir -p gpurun_out/r2
python -m pytest tests -m gpu -q -x ${PYTEST_ARGS:-} > gpurun_out/r2/pytest.log 2>&1; echo pytest_rc=$?
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2/smoke.log 2>&1; echo smoke_rc=$?
tail -3 gpurun_out/r2/pytest.log
