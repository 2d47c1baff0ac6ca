timeout 900 python -m pytest tests/test_gpu.py -x -q -k "perm" > gpurun_out/s29_tests.log 2>&1
SPTK_SORT_WIDE=1 timeout 900 python -m pytest tests/test_gpu.py -x -q -k "perm_bitexact" >> gpurun_out/s29_tests.log 2>&1
python tools/sort_ab.py nell2 "" "sort_wide=1" > gpurun_out/s29_sortab.log 2>&1
python tools/sort_ab.py delicious "" "sort_wide=1" >> gpurun_out/s29_sortab.log 2>&1
python tools/sort_ab.py lbnl "" "sort_wide=1" >> gpurun_out/s29_sortab.log 2>&1
