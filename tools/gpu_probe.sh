mkdir -p gpurun_out
( nproc; free -g; lscpu | head -20; nvidia-smi; df -h /tmp /root ) > gpurun_out/box.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/bench_r02_base.json 2> gpurun_out/bench_r02_base.err
echo rc=$?
