timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s11_tests.log 2>&1
for cfg in "lbnl 16 f64" "tiny 8 f64" "nell2 16 f64" "delicious 16 f64"; do
  python tools/als_sweep.py $cfg "" "gj_warp=0" 2>&1 | grep ms/iter
done > gpurun_out/s11_ab.log 2>&1
SPTK_SIDE_PRIO=0 python tools/als_sweep.py lbnl 16 f64 "" > gpurun_out/s11_ab_prio0.log 2>&1
SPTK_SIDE_PRIO=0 python tools/als_sweep.py tiny 8 f64 "" >> gpurun_out/s11_ab_prio0.log 2>&1
python tools/timeline.py tiny 8 20 > gpurun_out/s11_tl_tiny.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s11_tl_lbnl.log 2>&1
python tools/timeline.py nell2 16 6 > gpurun_out/s11_tl_nell2.log 2>&1
