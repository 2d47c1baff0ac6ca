timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s28_tests.log 2>&1
for r in 1 2; do
python tools/opt_sweep.py lbnl 16 f64 "" "run=16" 2>&1 | grep ms/mode
REPS=5 python tools/als_sweep.py lbnl 16 f64 "" "run=16" 2>&1 | grep ms/iter
done > gpurun_out/s28_ab.log 2>&1
python tools/opt_sweep.py delicious 16 f64 "" >> gpurun_out/s28_ab.log 2>&1
