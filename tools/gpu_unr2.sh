mkdir -p gpurun_out
for s in WD HP BS; do
timeout 600 python tools/ab_env.py GLB_GRAPH_UNROLL=1 GLB_GRAPH_UNROLL=2 GLB_GRAPH_UNROLL=4 GLB_NO_FUSED_CTL=1 --strategy $s --reps 9 >> gpurun_out/unr2.log 2>&1
done
timeout 600 python tools/ab_env.py GLB_GRAPH_UNROLL=1 GLB_GRAPH_UNROLL=2 GLB_GRAPH_UNROLL=4 GLB_NO_FUSED_CTL=1 --strategy WD --algo bfs --reps 9 >> gpurun_out/unr2.log 2>&1
true
