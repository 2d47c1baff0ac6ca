python -m pytest tests -m gpu -q -x -k "cp_als or smoke or deterministic" > gpurun_out/s65_tests.log 2>&1
o=gpurun_out/s65_ab.log; : > $o
for r in 1 2; do
  for lib in tools/abx/libprev.so paper_1809_09175_b200/libsptk.so; do
    echo "== $lib" >> $o
    SPTK_LIB=$lib REPS=5 ITERS=50 timeout 600 python tools/als_sweep.py lbnl 16 f64 "" >> $o 2>&1
    SPTK_LIB=$lib REPS=3 ITERS=10 timeout 600 python tools/als_sweep.py delicious 16 f64 "" >> $o 2>&1
  done
done
python tools/timeline.py lbnl 16 10 > gpurun_out/s65_tl_lbnl.log 2>&1
