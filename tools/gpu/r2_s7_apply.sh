timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s7_tests.log 2>&1
for cfg in "lbnl 16 f64" "delicious 16 f64" "nell2 16 f64" "tiny 8 f64"; do
  for L in tools/abx/libbase.so tools/abx/libW4.so; do
    echo "== $L $cfg"; SPTK_LIB=$L python tools/als_sweep.py $cfg "" 2>&1 | grep ms/iter
  done
  echo "== libsptk $cfg"; python tools/als_sweep.py $cfg "" "prezero=0" 2>&1 | grep ms/iter
done > gpurun_out/s7_ab.log 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/s7_lbnl_launches.csv python tools/als_probe.py lbnl 16 8 > gpurun_out/s7_lbnl_probe.log 2>&1
