# full GPU tier; cluster-loop phase trace and pre-check A/B on C3 BFS
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q --durations=5 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -n 3 gpurun_out/pytest_gpu.log
GRAPHLB_B200_LIB=_exp/trace.so timeout 300 python tools/small_trace.py --tags BS,EP,WD --algo bfs > gpurun_out/small_trace.log 2>&1
GRAPHLB_B200_LIB=_exp/trace.so timeout 300 python tools/small_trace.py --tags BS --algo sssp >> gpurun_out/small_trace.log 2>&1
cat gpurun_out/small_trace.log | sort | uniq -c | sort -rn | head -n 20
timeout 600 python tools/ab_libs.py paper_1711_00231_b200/libgraphlb_b200.so _exp/noprecheck.so --grid 4096 --algo bfs --strategy BS,EP,WD --reps 3 > gpurun_out/ab_noprecheck.log 2>&1
tail -n 8 gpurun_out/ab_noprecheck.log
