timeout 900 python -m pytest tests/test_gpu.py -x -q -k "perm" > gpurun_out/s5_tests.log 2>&1
python tools/sort_ab.py nell2 "" "sort_onesweep=1" "sort_v1=1" > gpurun_out/s5_sortab.log 2>&1
python tools/sort_ab.py lbnl "" "sort_onesweep=1" "sort_v1=1" >> gpurun_out/s5_sortab.log 2>&1
python tools/sort_ab.py delicious "" "sort_onesweep=1" "sort_v1=1" >> gpurun_out/s5_sortab.log 2>&1
REPS=1 ncu --set full --clock-control none -k regex:"radix_downsweep2|radix_onesweep|radix_hist_all" -c 6 -o gpurun_out/s5_sort python tools/sort_ab.py nell2 "" "sort_onesweep=1" > gpurun_out/s5_ncu.log 2>&1
ncu -i gpurun_out/s5_sort.ncu-rep --page raw --csv > gpurun_out/s5_sort_raw.csv 2>/dev/null
