mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/base.so variants/bl1.so --strategy WD --algo sssp --reps 9 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/base.so variants/bl1.so --strategy WD,HP --algo bfs --reps 7 2>&1 | tail -4
timeout 600 python tools/ab_libs.py variants/base.so variants/bl1.so --strategy WD --algo sssp --skewed --reps 7 2>&1 | tail -2
