timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded or window" > gpurun_out/s24_tests.log 2>&1
for r in 1 2; do
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "prezero=0" 2>&1 | grep ms/iter
python tools/als_sweep.py nell2 16 f64 "" "prezero=0" 2>&1 | grep ms/iter
REPS=7 python tools/als_sweep.py tiny 8 f64 "" "prezero=0" 2>&1 | grep ms/iter
done > gpurun_out/s24_ab.log 2>&1
python tools/als_sweep.py delicious 16 f64 "" "prezero=0" >> gpurun_out/s24_ab.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s24_tl_lbnl.log 2>&1
