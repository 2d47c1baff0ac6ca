timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s34_tests.log 2>&1
for r in 1 2; do
for L in paper_1809_09175_b200/libsptk.so tools/abx/libnoearly.so; do
  echo "== $L"
  SPTK_LIB=$L REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter
  SPTK_LIB=$L REPS=7 python tools/als_sweep.py tiny 8 f64 "" 2>&1 | grep ms/iter
  SPTK_LIB=$L python tools/als_sweep.py nell2 16 f64 "" 2>&1 | grep ms/iter
done; done > gpurun_out/s34_ab.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s34_tl_lbnl.log 2>&1
