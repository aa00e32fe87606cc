mkdir -p gpurun_out
timeout 600 ncu --metrics lts__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum -k regex:k_gather -c 6 ./_exp/gather_peak 22 26 > gpurun_out/ncu_gp.log 2>&1
true
