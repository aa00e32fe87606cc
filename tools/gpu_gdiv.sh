mkdir -p gpurun_out
timeout 600 python tools/loop_overhead.py --grid-div > gpurun_out/gdiv_loop.log 2>&1
for s in WD BS HP; do
timeout 600 python tools/ab_env.py GLB_GRAPH_GRID_DIV=1 GLB_GRAPH_GRID_DIV=2 GLB_GRAPH_GRID_DIV=4 --strategy $s --reps 7 >> gpurun_out/gdiv_c2.log 2>&1
done
for d in 1 2 4; do GLB_GRAPH_GRID_DIV=$d timeout 900 python tools/c3_breakdown.py --strategies BS,WD,HP > gpurun_out/gdiv_c3_$d.log 2>&1; done
true
