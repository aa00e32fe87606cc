# per-strategy cluster size: parity + A/B vs the previous build; ncu of the C5 HP compaction (host loop)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or grid or records or quirks or variants" > gpurun_out/c16b_parity.log 2>&1; echo "rc=$?" >> gpurun_out/c16b_parity.log
tail -n 2 gpurun_out/c16b_parity.log
timeout 900 python tools/ab_libs.py _exp/cur.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo bfs --strategy BS,EP,WD,NS,HP --reps 2 > gpurun_out/c16b_c3_bfs.log 2>&1
timeout 900 python tools/ab_libs.py _exp/cur.so paper_1711_00231_b200/libgraphlb_b200.so --grid 4096 --algo sssp --strategy BS,EP,WD,NS,HP --reps 1 > gpurun_out/c16b_c3_sssp.log 2>&1
timeout 600 python tools/ab_libs.py _exp/cur.so paper_1711_00231_b200/libgraphlb_b200.so --algo sssp --strategy WD,HP,EP --reps 5 > gpurun_out/c16b_c2_sssp.log 2>&1
timeout 600 python tools/ab_libs.py _exp/cur.so paper_1711_00231_b200/libgraphlb_b200.so --algo bfs --strategy WD,HP,EP --reps 5 > gpurun_out/c16b_c2_bfs.log 2>&1
for f in gpurun_out/c16b_*.log; do echo "== $f"; tail -n 10 $f; done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_tag_compact|k_hp_window" -s 20 -c 4 \
  -o gpurun_out/hp_c5_tag -f python tools/suite.py --configs C5 --tags HP --algos sssp --reps 1 --loop host --out gpurun_out/tmp_c5.json > gpurun_out/ncu_hp_c5.log 2>&1
ls -la gpurun_out/hp_c5_tag.ncu-rep
