mkdir -p gpurun_out
for alg in bfs sssp; do
timeout 600 python tools/ab_env.py GLB_SMALL_CTAS=8 GLB_SMALL_CTAS=16 --strategy NS --algo $alg --reps 7 > gpurun_out/ns16_c2_$alg.log 2>&1
done
for f in gpurun_out/ns16_*.log; do echo "== $f"; tail -n 4 $f; done
