mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or grid or variants" > gpurun_out/epc2_parity.log 2>&1; echo "rc=$?" >> gpurun_out/epc2_parity.log
tail -n 2 gpurun_out/epc2_parity.log
timeout 900 python tools/ab_libs.py _exp/pre_carry.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo bfs --strategy EP --reps 2 > gpurun_out/epc2_c3.log 2>&1
timeout 600 python tools/ab_libs.py _exp/pre_carry.so paper_1711_00231_b200/libgraphlb_b200.so --algo bfs --strategy EP --reps 5 > gpurun_out/epc2_c2.log 2>&1
for f in gpurun_out/epc2_c*.log; do echo "== $f"; tail -n 2 $f; done
