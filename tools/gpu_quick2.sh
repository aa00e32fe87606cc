#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 1500 python tools/suite.py --configs C2,C3,C1 --reps 2 > gpurun_out/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite.log
true
