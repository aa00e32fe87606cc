# cluster-loop changes: parity (grid + corpus), A/B vs the previous build on C3 BFS / SSSP, phase trace
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "grid or corpus or records or quirks" > gpurun_out/c3b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/c3b_parity.log
tail -n 2 gpurun_out/c3b_parity.log
timeout 900 python tools/ab_libs.py _exp/head.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo bfs --strategy BS,EP,WD,NS,HP --reps 3 > gpurun_out/c3b_ab_bfs.log 2>&1
tail -n 10 gpurun_out/c3b_ab_bfs.log
timeout 900 python tools/ab_libs.py _exp/head.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo sssp --strategy BS,EP --reps 2 > gpurun_out/c3b_ab_sssp.log 2>&1
tail -n 2 gpurun_out/c3b_ab_sssp.log
