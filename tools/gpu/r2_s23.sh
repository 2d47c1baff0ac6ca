for r in 1 2; do
for L in paper_1809_09175_b200/libsptk.so tools/abx/libM3P1.so tools/abx/libM3P2.so; do
  echo "== $L"; SPTK_LIB=$L REPS=5 python tools/als_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/iter
done
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "prezero=2" 2>&1 | grep ms/iter
done > gpurun_out/s23_ab.log 2>&1
for L in paper_1809_09175_b200/libsptk.so tools/abx/libM3P1.so; do
  echo "== $L"; SPTK_LIB=$L REPS=3 python tools/als_sweep.py delicious 16 f64 "" 2>&1 | grep ms/iter
done >> gpurun_out/s23_ab.log 2>&1
