mkdir -p gpurun_out
for algo in sssp bfs; do
  timeout 600 python tools/ab_libs.py _exp/fix.so:32 _exp/fix.so:24 --strategy BS,EP,WD,NS,HP --algo $algo --reps 5 >> gpurun_out/fix2_s22.log 2>&1
  timeout 600 python tools/ab_libs.py _exp/fix.so:32 _exp/fix.so:24 --strategy BS,EP,WD,HP --algo $algo --reps 5 --skewed >> gpurun_out/fix2_s22.log 2>&1
done
GRAPHLB_B200_LIB=_exp/fix.so timeout 1500 python tools/suite.py --configs C3 --reps 2 --out gpurun_out/suite_fix_c3.json > gpurun_out/suite_fix_c3.log 2>&1
true
GRAPHLB_B200_LIB=_exp/fix.so timeout 1500 python tools/suite.py --configs C3 --reps 2 --dist-bits 32 --out gpurun_out/suite_fix_c3_32.json > gpurun_out/suite_fix_c3_32.log 2>&1
true
