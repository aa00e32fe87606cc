mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/base.so variants/blwd.so variants/blall.so --strategy WD,HP,NS,BS --algo sssp --reps 5 2>&1 | tail -12
timeout 600 python tools/ab_libs.py variants/base.so variants/blwd.so variants/blall.so --strategy HP,NS,BS --algo bfs --reps 5 2>&1 | tail -9
timeout 600 python tools/ab_libs.py variants/base.so variants/blwd.so variants/blall.so --strategy HP,NS --algo sssp --skewed --reps 5 2>&1 | tail -6
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
