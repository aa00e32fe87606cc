mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_wd16.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_wd16.log
tail -n 2 gpurun_out/pytest_gpu_wd16.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_wd16.log 2>&1; tail -n 1 gpurun_out/smoke_wd16.log
timeout 1200 python tools/suite.py --configs C3,C2 --tags WD --reps 2 --out gpurun_out/suite_wd16.json > gpurun_out/suite_wd16.log 2>&1
grep "^|" gpurun_out/suite_wd16.log | grep -v 'cfg\|---'
