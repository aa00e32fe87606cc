mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 600 python tools/ab_libs.py variants/k4.so variants/k8m3.so variants/k8m2.so --strategy HP,NS --algo sssp --reps 5 2>&1 | tail -6
timeout 600 python tools/ab_libs.py variants/k4.so variants/k8m3.so variants/k8m2.so --strategy HP,NS --algo bfs --reps 5 2>&1 | tail -6
timeout 600 python tools/ab_libs.py variants/k4.so variants/k8m3.so variants/k8m2.so --strategy HP,NS --algo sssp --skewed --reps 5 2>&1 | tail -6
timeout 600 python tools/ab_libs.py variants/k4.so variants/k8m3.so variants/k8m2.so --strategy HP,NS --algo bfs --skewed --reps 5 2>&1 | tail -6
