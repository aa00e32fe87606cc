# ncu --set full of the cluster loop (C3 BFS EP, 16-CTA cluster) and of the BS compaction / relax on C3 SSSP
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_small_loop -c 1 \
  -o gpurun_out/c3_small_ep -f python tools/profile_grid.py --strategy EP --algo bfs > gpurun_out/ncu_c3_small.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bm_compact|k_bs_relax" -s 4000 -c 2 \
  -o gpurun_out/c3_bs_bm -f python tools/profile_grid.py --strategy BS --algo sssp > gpurun_out/ncu_c3_bm2.log 2>&1
ls -la gpurun_out/*.ncu-rep
