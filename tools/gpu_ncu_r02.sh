# round-2 ncu evidence: launch list of the bench command (host loop), --set full of
# k_wd_relax (C2 SSSP), k_hp_window + k_bigbin (C4 BFS), k_hp_window (C2 SSSP), peer exchange
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --e2e-steps 0 --loop host > gpurun_out/r02_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "glb traversal (host loop)/" \
  -k regex:k_wd_relax -s 1 -c 3 -o gpurun_out/r02_wd_relax -f \
  python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/r02_ncu_wd.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_hp_window|k_bigbin" -c 6 \
  -o gpurun_out/r02_hp_c4 -f python tools/profile_run.py --strategy HP --algo bfs --runs 1 --loop host --skewed > gpurun_out/r02_ncu_hp_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hp_window -s 2 -c 3 \
  -o gpurun_out/r02_hp_c2 -f python tools/profile_run.py --strategy HP --algo sssp --runs 1 --loop host > gpurun_out/r02_ncu_hp_c2.log 2>&1
ls -la gpurun_out/*.ncu-rep
true
