mkdir -p gpurun_out
GLB_CTRL_IN_BRANCH=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus and graph and default" > gpurun_out/inb_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/inb_pytest.log
for e in 0 1; do
  if [ $e = 1 ]; then export GLB_CTRL_IN_BRANCH=1; fi
  echo "== inb=$e" >> gpurun_out/inb_ab.log
  timeout 600 python tools/ab_libs.py _exp/inb.so --strategy BS,WD,HP --algo sssp --reps 5 >> gpurun_out/inb_ab.log 2>&1
  timeout 900 python tools/c3_breakdown.py --strategies BS,WD > gpurun_out/inb_c3_$e.log 2>&1
done
true
