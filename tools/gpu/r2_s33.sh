timeout 900 python -m pytest tests/test_gpu.py -q -k "cp_als_full_size" -v > gpurun_out/s33_tests.log 2>&1
for r in 1 2; do
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "apply_mma_rows=16384" 2>&1 | grep ms/iter
REPS=7 python tools/als_sweep.py tiny 8 f64 "" "apply_mma_rows=16384" 2>&1 | grep ms/iter
done > gpurun_out/s33_ab.log 2>&1
