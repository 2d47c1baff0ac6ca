for r in 1 2; do
for L in paper_1809_09175_b200/libsptk.so tools/abx/libtb48.so tools/abx/libtb64.so; do
  echo "== $L"; SPTK_LIB=$L REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter
done; done > gpurun_out/s43_ab.log 2>&1
