#!/bin/bash
# cfg2 narrow engine: 8x8-tile row-group weight gradient - tests, A/B (dev lib), bench line
mkdir -p gpurun_out/r2
timeout 900 python -m pytest tests/test_gpu_narrow.py tests/test_gpu_parity.py tests/test_gpu_edges.py -q -x > gpurun_out/r2/g4_pytest.log 2>&1; echo pytest_rc=$?
tail -3 gpurun_out/r2/g4_pytest.log
for v in 0 1 0 1; do echo "G4=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_G4=$v python scripts/narrow_probe.py cfg2 20 | tail -1; done
timeout 300 python bench.py --cfg cfg2 --steps 10 --warmup 3 > gpurun_out/r2/g4_cfg2.json 2> gpurun_out/r2/g4_cfg2.err; echo bench_rc=$?
tail -c 600 gpurun_out/r2/g4_cfg2.json
#!/bin/bash
for v in 0 1; do echo "G4=$v"; HMC_LIB=$PWD/paper_2507_14652_b200/libhmc_dev.so HMC_NW_G4=$v python scripts/narrow_phases.py cfg2 | tail -10; done
