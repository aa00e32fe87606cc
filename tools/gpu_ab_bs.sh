# BS: nodes per thread 1 / 2 / 4 on C3 SSSP + C2 SSSP/BFS, then parity of the default build
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/bs1.so variants/bs2.so variants/bs4.so --strategy BS --algo sssp --grid 4096 --reps 3 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/bs1.so variants/bs2.so variants/bs4.so --strategy BS --algo sssp --reps 5 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/bs1.so variants/bs2.so variants/bs4.so --strategy BS --algo bfs --grid 4096 --reps 3 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
