# HP id-ordered super-lists (k_tag_compact): parity + C5 A/B
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "corpus or renormalise or variants or quirks or hp or records" > gpurun_out/hpd_parity.log 2>&1; echo "rc=$?" >> gpurun_out/hpd_parity.log
tail -n 2 gpurun_out/hpd_parity.log
timeout 900 python tools/c5_env_probe.py GLB_WD_DENSE=0 GLB_WD_DENSE= --tags HP > gpurun_out/c5_hpdense.log 2>&1
tail -n 4 gpurun_out/c5_hpdense.log
