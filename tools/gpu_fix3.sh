mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for b in 32 24; do
GRAPHLB_B200_LIB=_exp/fix.so timeout 1200 python tools/suite.py --configs C5 --reps 2 --dist-bits $b --out gpurun_out/suite5_fix_$b.json > gpurun_out/suite5_fix_$b.log 2>&1
done
true
