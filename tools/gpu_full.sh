#!/bin/bash
# round evidence: tests, bench (ours + reference), suite C1-C4
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 1800 python tools/suite.py --configs C1,C2,C4,C3 --reps 2 > gpurun_out/suite.log 2>&1
true
