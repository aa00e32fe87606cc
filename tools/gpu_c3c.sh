# A/B (weighted walks keep the pre-check) + ncu --set full of the id-ordered BS relax and the compaction on C3 SSSP
mkdir -p gpurun_out
timeout 900 python tools/ab_libs.py _exp/head.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo sssp --strategy BS --reps 2 > gpurun_out/c3c_ab_sssp.log 2>&1
timeout 900 python tools/ab_libs.py _exp/head.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo bfs --strategy BS,NS --reps 2 > gpurun_out/c3c_ab_bfs.log 2>&1
tail -n 4 gpurun_out/c3c_ab_sssp.log gpurun_out/c3c_ab_bfs.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bs_relax -s 3000 -c 1 -o gpurun_out/c3_bs_relax python tools/profile_grid.py --strategy BS --algo sssp > gpurun_out/ncu_c3_bs.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_bm_compact -s 2000 -c 1 -o gpurun_out/c3_bm_compact python tools/profile_grid.py --strategy BS --algo sssp > gpurun_out/ncu_c3_bm.log 2>&1
ls -la gpurun_out/*.ncu-rep
