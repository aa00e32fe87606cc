#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python tools/suite.py --configs C1,C2,C4,C3 --reps 2 > gpurun_out/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite.log
true
