mkdir -p gpurun_out
for L in head n24; do
  GRAPHLB_B200_LIB=_exp/$L.so timeout 1500 python tools/suite.py --configs C2,C3,C4 --reps 3 --out gpurun_out/suite_$L.json > gpurun_out/suite_$L.log 2>&1
  GRAPHLB_B200_LIB=_exp/$L.so timeout 900 python tools/suite.py --configs C5 --reps 2 --out gpurun_out/suite5_$L.json > gpurun_out/suite5_$L.log 2>&1
done
true
