#!/bin/bash
mkdir -p gpurun_out
export GLB_BENCH_BACKEND=gloo
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 2 --warmup 1 --scale 18 > gpurun_out/shard2.log 2>&1; echo "rc=$?" >> gpurun_out/shard2.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 4 --steps 2 --warmup 1 --scale 18 --strategy HP --algo bfs > gpurun_out/shard4.log 2>&1; echo "rc=$?" >> gpurun_out/shard4.log
unset GLB_BENCH_BACKEND
timeout 900 python -m pytest tests -m gpu -x -q -k sharded > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
