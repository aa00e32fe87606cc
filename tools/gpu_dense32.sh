# dense WD scans / HP id-ordered super-lists in the 32-bit tier (C2, C4): A/B
mkdir -p gpurun_out
for alg in sssp bfs; do
timeout 600 python tools/ab_env.py GLB_WD_DENSE=0 GLB_WD_DENSE=1 --strategy HP --algo $alg --reps 5 > gpurun_out/d32_c2_hp_$alg.log 2>&1
timeout 600 python tools/ab_env.py GLB_WD_DENSE=0 GLB_WD_DENSE=1 --strategy HP --algo $alg --reps 5 --skewed > gpurun_out/d32_c4_hp_$alg.log 2>&1
timeout 600 python tools/ab_env.py GLB_WD_DENSE=0 GLB_WD_DENSE=1 --strategy WD --algo $alg --reps 5 --skewed > gpurun_out/d32_c4_wd_$alg.log 2>&1
done
for f in gpurun_out/d32_*.log; do echo "== $f"; tail -n 2 $f; done
