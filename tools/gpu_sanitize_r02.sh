# compute-sanitizer on the round-2 build: memcheck (full workload), racecheck + synccheck (--quick)
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 2400 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_run.py > gpurun_out/r02_sanitize_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02_sanitize_memcheck.log
GLB_NO_PDL=1 timeout 2400 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_run.py --quick > gpurun_out/r02_sanitize_racecheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02_sanitize_racecheck.log
timeout 2400 compute-sanitizer --tool synccheck --print-limit 20 python tools/sanitize_run.py --quick > gpurun_out/r02_sanitize_synccheck.log 2>&1; echo "rc=$?" >> gpurun_out/r02_sanitize_synccheck.log
for f in memcheck racecheck synccheck; do echo "== $f"; tail -4 gpurun_out/r02_sanitize_$f.log; done
