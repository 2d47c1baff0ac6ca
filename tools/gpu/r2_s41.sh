ncu --set full --clock-control none --import-source on -k regex:mttkrp_slice -c 3 -o gpurun_out/s41_nell2_slice python tools/als_probe.py nell2 16 2 > gpurun_out/s41_ncu1.log 2>&1
ncu -i gpurun_out/s41_nell2_slice.ncu-rep --page raw --csv > gpurun_out/s41_nell2_slice_raw.csv 2>/dev/null
ncu --set full --clock-control none -k regex:apply_gram_mma -s 4 -c 1 -o gpurun_out/s41_apply python tools/als_probe.py lbnl 16 3 > gpurun_out/s41_ncu2.log 2>&1
ncu -i gpurun_out/s41_apply.ncu-rep --page raw --csv > gpurun_out/s41_apply_raw.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/s41_lbnl_traffic.csv python tools/als_probe.py lbnl 16 3 > gpurun_out/s41_ncu3.log 2>&1
