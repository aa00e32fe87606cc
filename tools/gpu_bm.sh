# BS id-ordered frontiers: parity (threshold 1 and default) + A/B of the threshold on C3 / C2 / C4
mkdir -p gpurun_out
GLB_BM_THR=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/bm_parity_thr1.log 2>&1; echo "rc=$?" >> gpurun_out/bm_parity_thr1.log
tail -2 gpurun_out/bm_parity_thr1.log
V="GLB_BM_THR=0 GLB_BM_THR=16384 GLB_BM_THR=32768 GLB_BM_THR=65536"
timeout 900 python tools/ab_env.py $V --strategy BS --algo sssp --grid 4096 --reps 3 > gpurun_out/bm_ab_c3_sssp.log 2>&1
timeout 600 python tools/ab_env.py $V --strategy BS --algo sssp --reps 5 > gpurun_out/bm_ab_c2_sssp.log 2>&1
timeout 600 python tools/ab_env.py $V --strategy BS --algo bfs --reps 5 > gpurun_out/bm_ab_c2_bfs.log 2>&1
timeout 600 python tools/c3_sort_probe.py --env GLB_BM_THR --thr 32768 > gpurun_out/bm_probe.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_bm_compact -s 200 -c 20 --csv python tools/profile_grid.py --strategy BS --algo sssp > gpurun_out/bm_ncu.csv 2>&1
for f in gpurun_out/bm_ab_*.log; do echo "== $f"; tail -n 5 $f; done
cat gpurun_out/bm_probe.log
grep k_bm_compact gpurun_out/bm_ncu.csv | tail -n 5
