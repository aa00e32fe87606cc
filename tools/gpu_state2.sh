mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu2.log
tail -n 2 gpurun_out/pytest_gpu2.log
timeout 1200 python tools/suite.py --configs C5 --reps 2 --out gpurun_out/suite_c5_s2.json > gpurun_out/suite_c5_s2.log 2>&1
timeout 2400 python tools/suite.py --configs C2,C4,C3 --reps 2 --out gpurun_out/suite_s2.json > gpurun_out/suite_s2.log 2>&1
grep "^|" gpurun_out/suite_s2.log | tail -n 30; grep "^|" gpurun_out/suite_c5_s2.log | tail -n 10
