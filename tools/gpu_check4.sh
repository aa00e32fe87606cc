mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest tests/test_summaries.py tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/head4.so --dist-bits 24 --strategy WD,HP --algo sssp --reps 5 2>&1 | tail -2
timeout 600 python tools/ab_libs.py variants/head4.so --dist-bits 32 --strategy WD,HP --algo sssp --reps 5 2>&1 | tail -2
timeout 300 python tools/profile_run.py --strategy HP --algo sssp --runs 2 --loop graph --records 2>&1 | tail -62 > gpurun_out/rec_hp_graph.txt
head -40 gpurun_out/rec_hp_graph.txt
