#!/bin/bash
mkdir -p gpurun_out/mwg
python -m pytest tests -m gpu -q > gpurun_out/mwg/pytest_all.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/mwg/pytest_all.log
for c in cfg3 cfg4 cfg5; do python -c "
import sys; sys.path.insert(0,'.')
from hmcdata import make_problem
from paper_2507_14652_b200 import abi
p=make_problem('$c'); c=abi.Context(p); print('$c', abi.hmc_engine_info(c.ctx))"; done
