timeout 900 python -m pytest tests/test_gpu.py -x -q -k "perm" > gpurun_out/s6_tests.log 2>&1
python tools/sort_ab.py nell2 "" "sort_pipe=1" "sort_v1=1" > gpurun_out/s6_sortab.log 2>&1
python tools/sort_ab.py lbnl "" "sort_pipe=1" >> gpurun_out/s6_sortab.log 2>&1
python tools/sort_ab.py delicious "" "sort_pipe=1" >> gpurun_out/s6_sortab.log 2>&1
REPS=1 ncu --set full --clock-control none -k regex:"radix_downsweep_pipe" -c 2 -o gpurun_out/s6_pipe python tools/sort_ab.py nell2 "sort_pipe=1" > gpurun_out/s6_ncu.log 2>&1
ncu -i gpurun_out/s6_pipe.ncu-rep --page raw --csv > gpurun_out/s6_pipe_raw.csv 2>/dev/null
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/s6_lbnl_launches.csv python tools/als_probe.py lbnl 16 8 > gpurun_out/s6_lbnl_probe.log 2>&1
python tools/als_sweep.py lbnl 16 f64 "" > gpurun_out/s6_lbnl_als.log 2>&1
