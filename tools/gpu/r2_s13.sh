timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s13_tests.log 2>&1
for r in 1 2; do
for cfg in "tiny 8 f64" "lbnl 16 f64"; do
  REPS=7 python tools/als_sweep.py $cfg "" "prezero=0" "gj_warp=0" 2>&1 | grep ms/iter
done; done > gpurun_out/s13_ab.log 2>&1
python tools/timeline.py tiny 8 20 > gpurun_out/s13_tl_tiny.log 2>&1
python tools/timeline.py tiny 8 20 "prezero=0" > gpurun_out/s13_tl_tiny_pz0.log 2>&1
