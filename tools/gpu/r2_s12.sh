timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s12_tests.log 2>&1
for cfg in "tiny 8 f64" "lbnl 16 f64" "nell2 16 f64" "delicious 16 f64"; do
  python tools/als_sweep.py $cfg "" "gj_warp=0" 2>&1 | grep ms/iter
done > gpurun_out/s12_ab.log 2>&1
for p in 0 1; do SPTK_SIDE_PRIO=$p python tools/als_sweep.py tiny 8 f64 "" "gj_warp=0" 2>&1 | grep ms/iter | sed "s/^/prio=$p /"; done >> gpurun_out/s12_ab.log 2>&1
python tools/timeline.py tiny 8 20 > gpurun_out/s12_tl_tiny.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s12_tl_lbnl.log 2>&1
