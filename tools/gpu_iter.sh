# iterate: build, GPU parity suite, then the C2/C4 strategy table (argument: extra pytest -k filter)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest tests -m gpu -x -q ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 900 python tools/suite.py --configs ${SUITE_CFGS:-C2,C4} --tags ${SUITE_TAGS:-WD,NS,HP} --reps 3 --out gpurun_out/suite.json > gpurun_out/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite.log
tail -25 gpurun_out/suite.log
