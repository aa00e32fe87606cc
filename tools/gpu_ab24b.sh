mkdir -p gpurun_out
for algo in sssp bfs; do
  timeout 600 python tools/ab_records.py _exp/head.so _exp/n24.so --strategy WD --algo $algo > gpurun_out/ab24_rec_$algo.log 2>&1
done
timeout 600 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy WD --algo sssp --dist-bits 32 --reps 5 > gpurun_out/ab24_d32.log 2>&1
GLB_NO_SMALL=1 timeout 600 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy WD --algo sssp --reps 5 > gpurun_out/ab24_nosmall.log 2>&1
timeout 600 python tools/ab_libs.py _exp/head.so _exp/n24.so --strategy WD --algo sssp --loop host --reps 5 > gpurun_out/ab24_host.log 2>&1
true
