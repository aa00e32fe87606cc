# HP/NS adaptive warp chunks: parity, suite C2/C3/C4, HP records
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_parity.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_parity.log
tail -3 gpurun_out/pytest_parity.log
timeout 900 python tools/suite.py --configs ${SUITE_CFGS:-C2,C4,C3} --tags ${SUITE_TAGS:-NS,HP,WD} --reps 3 --out gpurun_out/suite3.json > gpurun_out/suite3.log 2>&1; echo "suite rc=$?" >> gpurun_out/suite3.log
grep "^|" gpurun_out/suite3.log | tail -26
timeout 300 python tools/profile_run.py --strategy HP --algo sssp --runs 2 --loop host --records > gpurun_out/rec_hp_c2.txt 2>&1
true
