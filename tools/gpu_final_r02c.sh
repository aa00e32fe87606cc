#!/bin/bash
# round-2 (session 3) evidence on the committed build: GPU tier, smoke, bench (ours + reference),
# ncu launch list + --set full of k_wd_relax and of the C5 HP tag compaction / window kernels, suite C1-C5
# (compute-sanitizer is closed on this pool)
O=gpurun_out/final
rm -rf $O; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || exit 1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err
timeout 900 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --e2e-steps 0 --loop host > $O/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 1 -c 3 \
  -o $O/wd_relax_full -f python tools/profile_run.py --strategy WD --algo sssp --loop host --runs 1 > $O/ncu_full.log 2>&1
timeout 2400 python tools/suite.py --configs C1,C2,C4,C3 --reps 3 --out $O/suite.json > $O/suite.log 2>&1
timeout 1500 python tools/suite.py --configs C5 --reps 2 --out $O/suite_c5.json > $O/suite_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tag_compact|k_hp_window" -s 20 -c 4 \
  -o $O/hp_c5_tag -f python tools/suite.py --configs C5 --tags HP --algos sssp --reps 1 --loop host --out $O/tmp_c5.json > $O/ncu_hp_c5.log 2>&1
tail -n 2 $O/pytest_gpu.log; tail -n 1 $O/smoke.log; head -c 400 $O/bench.json; echo; grep "^|" $O/suite.log | tail -n 40; grep "^|" $O/suite_c5.log | tail -n 10
