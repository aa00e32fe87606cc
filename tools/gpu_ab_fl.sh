mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/fl0.so variants/fl1.so --strategy BS --algo sssp --grid 4096 --reps 3 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/fl0.so variants/fl1.so --strategy BS --algo sssp --reps 5 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/fl0.so variants/fl1.so --strategy BS --algo bfs --reps 5 2>&1 | tail -2
