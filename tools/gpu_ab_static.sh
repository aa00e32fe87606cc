mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/own512b.so variants/static1.so --strategy HP,NS --algo sssp --reps 5 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/own512b.so variants/static1.so --strategy HP,NS --algo bfs --reps 5 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/own512b.so variants/static1.so --strategy HP,NS --algo sssp --skewed --reps 5 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "corpus or random or c2 or hp" > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
