mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/head.so variants/m3.so variants/e4m3b.so variants/e4m4b.so --strategy WD --algo sssp --reps 7 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/head.so variants/m3.so variants/e4m3b.so variants/e4m4b.so --strategy WD --algo bfs --reps 7 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/head.so variants/m3.so variants/e4m3b.so variants/e4m4b.so --strategy WD --algo sssp --skewed --reps 7 2>&1 | tail -4
