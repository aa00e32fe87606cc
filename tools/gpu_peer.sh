# peer-memory sharded path: GPU tests + sharded bench (2 ranks sharing one GPU, IPC)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_peer.py tests/test_gpu_parity.py -k "peer or sharded" -x -q --durations=10 > gpurun_out/pytest_peer.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_peer.log
tail -25 gpurun_out/pytest_peer.log
timeout 600 python bench.py --gpus 2 --scale 20 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_g2_peer.json 2> gpurun_out/bench_g2_peer.err; echo "rc=$?" >> gpurun_out/bench_g2_peer.err
tail -3 gpurun_out/bench_g2_peer.err; cat gpurun_out/bench_g2_peer.json
timeout 600 python bench.py --gpus 2 --scale 20 --steps 3 --warmup 3 --no-cpu --transport torch > gpurun_out/bench_g2_torch.json 2> gpurun_out/bench_g2_torch.err; echo "rc=$?" >> gpurun_out/bench_g2_torch.err
tail -3 gpurun_out/bench_g2_torch.err; cat gpurun_out/bench_g2_torch.json
