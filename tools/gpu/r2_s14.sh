python tools/opt_sweep.py delicious 16 f64 "" "big_first=256" "big_first=1024" > gpurun_out/s14_big.log 2>&1
python tools/opt_sweep.py amazon 16 f64 "" "big_first=256" >> gpurun_out/s14_big.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s14_tests.log 2>&1
python tools/timeline.py tiny 8 20 > gpurun_out/s14_tl_tiny.log 2>&1
