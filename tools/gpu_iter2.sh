# HP/NS single-kernel steps + WD variants: parity, suite, A/B, HP records
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
timeout 900 python tools/suite.py --configs C2,C3,C4 --tags BS,NS,HP,WD --reps 3 --out gpurun_out/suite2.json > gpurun_out/suite2.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite2.log
grep "^|" gpurun_out/suite2.log | tail -26
timeout 600 python tools/ab_libs.py variants/base.so variants/e4m3.so variants/e4m4.so --strategy WD --algo sssp --reps 7 > gpurun_out/ab_wd.log 2>&1; tail -8 gpurun_out/ab_wd.log
timeout 600 python tools/ab_env.py GLB_NONE=1 GLB_L2_PERSIST=1 --strategy WD --algo sssp --reps 7 > gpurun_out/ab_l2.log 2>&1; tail -4 gpurun_out/ab_l2.log
timeout 300 python tools/profile_run.py --strategy HP,WD --algo sssp --runs 2 --loop host --records > gpurun_out/rec_hp_c2.txt 2>&1
true
