mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -m paper_1711_00231_b200 --gen rmat --scale 22 --edge-factor 16 --algo sssp --verify --loop graph --out gpurun_out/cli_c2.csv > gpurun_out/cli_c2.log 2>&1; echo "rc=$?" >> gpurun_out/cli_c2.log
true
