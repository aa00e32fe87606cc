# 16-CTA (non-portable) cluster loop vs 8: C3 BFS / SSSP, C2 tails
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py _exp/cur.so _exp/c16.so --grid 4096 --algo bfs --strategy BS,EP,WD,NS,HP --reps 2 > gpurun_out/c16_c3_bfs.log 2>&1
timeout 900 python tools/ab_libs.py _exp/cur.so _exp/c16.so --grid 4096 --algo sssp --strategy BS,NS --reps 2 > gpurun_out/c16_c3_sssp.log 2>&1
timeout 600 python tools/ab_libs.py _exp/cur.so _exp/c16.so --algo sssp --strategy WD,HP --reps 5 > gpurun_out/c16_c2_sssp.log 2>&1
for f in gpurun_out/c16_*.log; do echo "== $f"; tail -n 10 $f; done
