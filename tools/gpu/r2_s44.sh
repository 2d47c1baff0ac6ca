for r in 1 2; do
for L in paper_1809_09175_b200/libsptk.so tools/abx/libn5u1m3.so tools/abx/libn5u2m3.so; do
  echo "== $L"; SPTK_LIB=$L python tools/opt_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/mode; SPTK_LIB=$L REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter
done; done > gpurun_out/s44_ab.log 2>&1
