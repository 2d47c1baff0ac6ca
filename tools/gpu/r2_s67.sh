REPS=5 ITERS=50 timeout 600 python tools/als_sweep.py lbnl 16 f64 "" "prezero_mb=100" "prezero_mb=64" "" "prezero_mb=100" > gpurun_out/s67_ab.log 2>&1
REPS=3 ITERS=10 timeout 900 python tools/als_sweep.py delicious 16 f64 "" "prezero_mb=64" "" "prezero_mb=64" >> gpurun_out/s67_ab.log 2>&1
python tools/timeline.py lbnl 16 10 f64 prezero_mb=100 > gpurun_out/s67_tl_lbnl.log 2>&1
