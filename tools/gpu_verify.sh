#!/bin/bash
# tests + smoke + a short bench on the committed build
mkdir -p gpurun_out/verify
O=gpurun_out/verify
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $O/smoke.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-extras > $O/bench.log 2>&1
true
