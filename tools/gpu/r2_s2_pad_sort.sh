python tools/sort_ab.py nell2 "" "sort_v1=1" > gpurun_out/s3_sort_nell2.log 2>&1
python tools/sort_ab.py lbnl "" "sort_v1=1" > gpurun_out/s3_sort_lbnl.log 2>&1
python tools/sort_ab.py delicious "" "sort_v1=1" > gpurun_out/s3_sort_delicious.log 2>&1
python tools/als_sweep.py nell2 16 f64 "" > gpurun_out/s3_als_r16.log 2>&1
python tools/als_sweep.py nell2 17 f64 "" "pad_rank=0" "pad_rank=8" "pad_rank=16" > gpurun_out/s3_als_r17.log 2>&1
python tools/als_sweep.py nell2 10 f64 "" "pad_rank=0" > gpurun_out/s3_als_r10.log 2>&1
python tools/als_sweep.py nell2 12 f32 "" "pad_rank=0" > gpurun_out/s3_als_r12f32.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s3_tests.log 2>&1
