mkdir -p gpurun_out
nproc > gpurun_out/host_bw.log; lscpu | grep -i "model name\|socket\|numa\|^CPU(s)" >> gpurun_out/host_bw.log
./_exp/host_bw >> gpurun_out/host_bw.log 2>&1
true
