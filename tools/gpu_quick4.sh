#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/profile_run.py --strategy WD --algo sssp --runs 2 --loop graph --records > gpurun_out/records_graph.log 2>&1
timeout 600 python bench.py --no-extras > gpurun_out/bench.log 2>&1
true
