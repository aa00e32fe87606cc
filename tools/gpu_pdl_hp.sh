# PDL between the BS compaction and relax: parity + A/B; ncu --set full of the HP kernels on the current build
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "grid or corpus or quirks or variants" > gpurun_out/pdl_parity.log 2>&1; echo "rc=$?" >> gpurun_out/pdl_parity.log
tail -n 2 gpurun_out/pdl_parity.log
timeout 900 python tools/ab_env.py GLB_NO_PDL=1 GLB_NO_PDL= --strategy BS --algo sssp --grid 4096 --reps 2 > gpurun_out/pdl_ab_c3.log 2>&1
timeout 600 python tools/ab_env.py GLB_NO_PDL=1 GLB_NO_PDL= --strategy BS --algo sssp --reps 5 > gpurun_out/pdl_ab_c2.log 2>&1
tail -n 3 gpurun_out/pdl_ab_c3.log gpurun_out/pdl_ab_c2.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hp_window|k_bigbin" -c 6 \
  -o gpurun_out/r02c_hp_c4 -f python tools/profile_run.py --strategy HP --algo bfs --runs 1 --loop host --skewed > gpurun_out/r02c_ncu_hp_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hp_window -s 2 -c 3 \
  -o gpurun_out/r02c_hp_c2 -f python tools/profile_run.py --strategy HP --algo sssp --runs 1 --loop host > gpurun_out/r02c_ncu_hp_c2.log 2>&1
timeout 600 python tools/e2e_probe.py --loop graph --reps 4 > gpurun_out/e2e_probe.log 2>&1
cat gpurun_out/e2e_probe.log | tail -n 4
ls -la gpurun_out/*.ncu-rep
