#!/bin/bash
# narrow engine fused top layer (cfg2): tests, A/B (dev lib HMC_NW_FUSE), phases, bench line
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/r2/fuse_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2/fuse_pytest.log
for v in 0 1 0 1; do echo "FUSE=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_FUSE=$v python scripts/narrow_probe.py cfg2 20 | tail -1; done
for v in 0 1; do echo "FUSE=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_FUSE=$v python scripts/narrow_phases.py cfg2 | tail -10; done
timeout 300 python bench.py --cfg cfg2 --steps 10 --warmup 3 > gpurun_out/r2/fuse_cfg2.json 2> gpurun_out/r2/fuse_cfg2.err; echo bench_rc=$?
python -c "import json; d=json.loads(open('gpurun_out/r2/fuse_cfg2.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'])"
