# dense WD scans in the 24-bit tier: parity + C5 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or renormalise or variants or quirks or c2 or 24bit" > gpurun_out/d24_parity.log 2>&1; echo "rc=$?" >> gpurun_out/d24_parity.log
tail -n 2 gpurun_out/d24_parity.log
timeout 900 python tools/c5_dense_probe.py --bits 0 > gpurun_out/c5_dense24.log 2>&1
tail -n 4 gpurun_out/c5_dense24.log
timeout 900 python tests/../tools/suite.py --configs C5 --reps 1 --out gpurun_out/suite_c5_d24.json > gpurun_out/suite_c5_d24.log 2>&1
grep "^|" gpurun_out/suite_c5_d24.log | tail -n 10
