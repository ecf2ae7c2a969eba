#!/bin/bash
# DATA-mode checks on one GPU: world-1 NCCL tests, emulated ranks, and the bench's data-mode line
# through torchrun with one process (the path the 8-GPU SCALE run takes)
mkdir -p gpurun_out/r2
python -m pytest tests/test_gpu_datamode.py tests/test_gpu_shard_emulation.py -q -x 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29517 \
  bench.py --gpus 1 --steps 5 --warmup 3 --parallel data --no-cpu-baseline --breakdown > gpurun_out/r2/bench_cfg5_data1.json 2> gpurun_out/r2/bench_cfg5_data1.err
echo torchrun_rc=$?
tail -c 1500 gpurun_out/r2/bench_cfg5_data1.json; grep -c "NCCL INFO" gpurun_out/r2/bench_cfg5_data1.json gpurun_out/r2/bench_cfg5_data1.err; tail -12 gpurun_out/r2/bench_cfg5_data1.err
