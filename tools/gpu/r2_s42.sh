timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s42_tests.log 2>&1
for r in 1 2; do
for L in tools/abx/libbase.so paper_1809_09175_b200/libsptk.so; do
  echo "== $L"
  SPTK_LIB=$L REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter
  SPTK_LIB=$L REPS=3 python tools/als_sweep.py delicious 16 f64 "" 2>&1 | grep ms/iter
  SPTK_LIB=$L REPS=3 python tools/als_sweep.py nell2 16 f64 "" 2>&1 | grep ms/iter
done; done > gpurun_out/s42_ab.log 2>&1
ncu --set full --clock-control none -k regex:apply_gram_mma -s 4 -c 1 -o gpurun_out/s42_apply python tools/als_probe.py lbnl 16 3 > gpurun_out/s42_ncu.log 2>&1
ncu -i gpurun_out/s42_apply.ncu-rep --page raw --csv > gpurun_out/s42_apply_raw.csv 2>/dev/null
