mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/blB.so variants/blC.so --strategy WD --algo sssp --reps 9 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/blB.so variants/blC.so --strategy WD --algo bfs --reps 9 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/blB.so variants/blC.so --strategy WD --algo sssp --skewed --reps 7 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "corpus or c2 or random or 24bit or dist_bits" > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
