# NS id-ordered frontiers: parity + A/B against the previous build on C2 / C3 / C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "grid or corpus or quirks or variants or c2" > gpurun_out/ns_parity.log 2>&1; echo "rc=$?" >> gpurun_out/ns_parity.log
tail -n 2 gpurun_out/ns_parity.log
timeout 600 python tools/ab_libs.py _exp/prens.so paper_1711_00231_b200/libgraphlb_b200.so --strategy NS,BS --algo bfs --reps 5 > gpurun_out/ns_ab_c2_bfs.log 2>&1
timeout 600 python tools/ab_libs.py _exp/prens.so paper_1711_00231_b200/libgraphlb_b200.so --strategy NS --algo sssp --reps 5 > gpurun_out/ns_ab_c2_sssp.log 2>&1
timeout 600 python tools/ab_libs.py _exp/prens.so paper_1711_00231_b200/libgraphlb_b200.so --strategy NS --algo sssp --skewed --reps 3 > gpurun_out/ns_ab_c4_sssp.log 2>&1
timeout 900 python tools/ab_libs.py _exp/prens.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --strategy NS --algo sssp --reps 2 > gpurun_out/ns_ab_c3_sssp.log 2>&1
timeout 900 python tools/ab_libs.py _exp/prens.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --strategy NS --algo bfs --reps 2 > gpurun_out/ns_ab_c3_bfs.log 2>&1
for f in gpurun_out/ns_ab_*.log; do echo "== $f"; tail -n 4 $f; done
