timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s21_tests.log 2>&1
for r in 1 2; do
for cfg in "lbnl 16 f64" "nell2 16 f64" "delicious 16 f64"; do
  python tools/als_sweep.py $cfg "" "fused_reduce=0" 2>&1 | grep ms/iter
done; done > gpurun_out/s21_ab.log 2>&1
python tools/timeline.py nell2 16 6 > gpurun_out/s21_tl_nell2.log 2>&1
