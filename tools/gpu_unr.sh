mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus and graph and default" > gpurun_out/unr_quick.log 2>&1; echo "rc=$?" >> gpurun_out/unr_quick.log
if grep -q "rc=0" gpurun_out/unr_quick.log; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  for u in 1 4; do
    export GLB_GRAPH_UNROLL=$u
    echo "== unroll=$u" >> gpurun_out/unr_ab.log
    timeout 600 python tools/ab_libs.py _exp/unr.so --strategy BS,EP,WD,NS,HP --algo sssp --reps 5 >> gpurun_out/unr_ab.log 2>&1
    timeout 600 python tools/ab_libs.py _exp/unr.so --strategy WD,HP --algo bfs --reps 5 >> gpurun_out/unr_ab.log 2>&1
    timeout 900 python tools/c3_breakdown.py --strategies BS,WD,HP > gpurun_out/unr_c3_$u.log 2>&1
    timeout 900 python tools/c3_breakdown.py --strategies BS,EP,WD --algo bfs > gpurun_out/unr_c3b_$u.log 2>&1
  done
fi
true
