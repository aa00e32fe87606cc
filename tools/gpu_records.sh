# per-launch records of HP vs WD (C2 SSSP, C4 BFS/SSSP) + ncu launch list of HP on C4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for loop in host graph; do
python tools/profile_run.py --strategy WD,HP,NS --algo sssp --runs 2 --loop $loop --records > gpurun_out/rec_c2_sssp_$loop.txt 2>&1
python tools/profile_run.py --strategy WD,HP,NS --algo bfs --runs 2 --skewed --loop $loop --records > gpurun_out/rec_c4_bfs_$loop.txt 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_hp.csv python tools/profile_run.py --strategy HP,WD --algo bfs --runs 1 --skewed --loop host > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_hp.csv python tools/profile_run.py --strategy HP,WD --algo sssp --runs 1 --loop host > /dev/null 2>&1
true
