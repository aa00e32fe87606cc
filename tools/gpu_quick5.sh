#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
python tools/ab_libs.py _exp/v4.so _exp/fused.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab.log 2>&1
python tools/ab_libs.py _exp/v4.so _exp/fused.so --strategy WD --algo bfs --reps 5 >> gpurun_out/ab.log 2>&1
timeout 900 python tools/suite.py --configs C3,C4 --reps 1 --tags WD,BS,HP > gpurun_out/suite.log 2>&1
true
