timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als" > gpurun_out/s19_tests.log 2>&1
for r in 1 2; do
SPTK_LIB=tools/abx/libbase.so REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter | sed 's/^/base /'
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "tail_blocks=16" "tail_blocks=8" 2>&1 | grep ms/iter
done > gpurun_out/s19_ab.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s19_tl_lbnl.log 2>&1
python tools/timeline.py lbnl 16 10 "tail_blocks=8" > gpurun_out/s19_tl_lbnl_tb8.log 2>&1
