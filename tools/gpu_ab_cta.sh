mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for algo in bfs sssp; do
timeout 600 python tools/ab_libs.py variants/cta512.so variants/own256.so variants/own512.so variants/own1024.so --strategy HP,NS --algo $algo --skewed --reps 5 2>&1 | tail -8
done
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -2 gpurun_out/pytest_parity.log
