#!/bin/bash
# quick GPU iteration: parity tests + e2e probe + bench lines (host and graph loop)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python tools/e2e_probe.py --loop graph > gpurun_out/e2e_probe.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --no-extras --no-cpu --loop host > gpurun_out/bench_host.log 2>&1
timeout 300 python tools/profile_run.py --strategy WD,HP --algo sssp --runs 2 --loop host --records > gpurun_out/records_sssp.log 2>&1
true
