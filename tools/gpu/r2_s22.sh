timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s22_tests.log 2>&1
for r in 1 2; do
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "apply_cluster=16" "apply_cluster=0" 2>&1 | grep ms/iter
REPS=7 python tools/als_sweep.py tiny 8 f64 "" "apply_cluster=0" 2>&1 | grep ms/iter
done > gpurun_out/s22_ab.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s22_tl_lbnl.log 2>&1
python tools/timeline.py tiny 8 20 > gpurun_out/s22_tl_tiny.log 2>&1
