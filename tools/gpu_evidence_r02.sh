# round-2 evidence on HEAD: bench (ours + reference), suite C1-C5, ncu launch list + --set full of k_wd_relax
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "rc=$?" >> gpurun_out/bench_ref.err
timeout 1800 python tools/suite.py --configs C1,C2,C4,C3,C5 --reps 3 --out gpurun_out/suite_all.json > gpurun_out/suite_all.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite_all.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --e2e-steps 0 --loop host > gpurun_out/r02_launch_bench.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 1 -c 3 -o gpurun_out/r02_wd_relax_final -f \
  python tools/profile_run.py --strategy WD --algo sssp --runs 1 --loop host > gpurun_out/r02_ncu_wd2.log 2>&1
grep "^|" gpurun_out/suite_all.log | tail -48
