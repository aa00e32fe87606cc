# round-2 final evidence on HEAD: GPU tier, smoke, bench (ours + reference), suite C1-C5
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 1800 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 1800 python tools/suite.py --configs C1,C2,C4,C3,C5 --reps 3 --out gpurun_out/suite_all.json > gpurun_out/suite_all.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite_all.log
tail -3 gpurun_out/pytest_gpu.log; tail -1 gpurun_out/smoke.log; grep "^|" gpurun_out/suite_all.log | tail -48
