mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus and graph and default" > gpurun_out/fctl_quick.log 2>&1; echo "rc=$?" >> gpurun_out/fctl_quick.log
if grep -q "rc=0" gpurun_out/fctl_quick.log; then
  timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
  for e in 1 0; do
    if [ $e = 1 ]; then export GLB_NO_FUSED_CTL=1; else unset GLB_NO_FUSED_CTL; fi
    echo "== nofused=$e" >> gpurun_out/fctl_ab.log
    timeout 600 python tools/ab_libs.py _exp/fctl.so --strategy BS,EP,WD,NS,HP --algo sssp --reps 5 >> gpurun_out/fctl_ab.log 2>&1
    timeout 600 python tools/ab_libs.py _exp/fctl.so --strategy BS,EP,WD,NS,HP --algo bfs --reps 5 >> gpurun_out/fctl_ab.log 2>&1
    timeout 900 python tools/c3_breakdown.py --strategies BS,WD,HP > gpurun_out/fctl_c3_$e.log 2>&1
  done
fi
true
