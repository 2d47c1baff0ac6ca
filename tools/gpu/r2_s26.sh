for r in 1 2; do
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "tail_rows=0" "tail_rows=2048" 2>&1 | grep ms/iter
REPS=7 python tools/als_sweep.py tiny 8 f64 "" "tail_rows=0" 2>&1 | grep ms/iter
python tools/als_sweep.py nell2 16 f64 "" "tail_rows=65536" 2>&1 | grep ms/iter
done > gpurun_out/s26_ab.log 2>&1
