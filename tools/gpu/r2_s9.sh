for cfg in "lbnl 16 f64" "delicious 16 f64"; do
  for L in paper_1809_09175_b200/libsptk.so tools/abx/libM3P2.so tools/abx/libM3P1.so; do
    echo "== $L $cfg"; SPTK_LIB=$L python tools/als_sweep.py $cfg "" 2>&1 | grep ms/iter
  done
done > gpurun_out/s9_ab.log 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/s9_lbnl_launches.csv python tools/als_probe.py lbnl 16 8 > gpurun_out/s9_lbnl_probe.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s9_tests.log 2>&1
