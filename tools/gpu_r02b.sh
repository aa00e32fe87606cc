# round-2 state check on HEAD: GPU tests, smoke, bench (ours), suite C2/C3/C4 all strategies
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 1200 python tools/suite.py --configs C2,C3,C4 --reps 3 --out gpurun_out/suite.json > gpurun_out/suite.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite.log
tail -40 gpurun_out/suite.log
