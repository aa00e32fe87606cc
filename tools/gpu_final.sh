#!/bin/bash
# round-end evidence: tests, smoke, bench (ours + reference), launch list,
# ncu --set full of the dominant kernel, suite C1-C5
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-extras --no-cpu --e2e-steps 0 > $O/ncu_launch_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_wd_relax -s 1 -c 2 \
  -o $O/wd_relax_full -f python tools/profile_run.py --strategy WD --algo sssp --loop host --runs 1 > $O/ncu_full.log 2>&1
timeout 2400 python tools/suite.py --configs C1,C2,C4,C3 --reps 2 --out $O/suite.json > $O/suite.log 2>&1
timeout 1200 python tools/suite.py --configs C5 --reps 2 --out $O/suite_c5.json > $O/suite_c5.log 2>&1
true
