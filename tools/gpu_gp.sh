mkdir -p gpurun_out
./_exp/gather_peak 22 26 > gpurun_out/gather_peak.log 2>&1
true
