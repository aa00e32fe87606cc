mkdir -p gpurun_out
for L in head n24; do
  GRAPHLB_B200_LIB=_exp/$L.so timeout 900 ncu --set full --clock-control none -k regex:k_wd_relax -c 8 \
    -o gpurun_out/ncu_wd_$L -f python tools/profile_run.py --strategy WD --algo sssp --scale 22 --runs 1 --loop host > gpurun_out/ncu_$L.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q -k "24bit or overflow or corpus" > gpurun_out/pytest_gpu24.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu24.log
true
