mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/blwd.so variants/blall2.so --strategy BS,HP,NS,WD --algo sssp --reps 5 2>&1 | tail -8
timeout 900 python tools/ab_libs.py variants/blall2.so variants/smbl.so --strategy BS,WD,HP --algo bfs --grid 4096 --reps 3 2>&1 | tail -6
timeout 900 python tools/ab_libs.py variants/blall2.so variants/smbl.so --strategy BS,WD --algo sssp --grid 4096 --reps 2 2>&1 | tail -4
