mkdir -p gpurun_out
timeout 300 python tools/e2e_probe.py --loop graph --reps 5 > gpurun_out/e2e_probe.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
true
