timeout 1200 python -m pytest tests/test_gpu_exact.py -x -q -k "lbnl or tiny" > gpurun_out/s20_tests.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "config or slice" >> gpurun_out/s20_tests.log 2>&1
for r in 1 2; do
python tools/opt_sweep.py lbnl 16 f64 "" "slice_fill=0" 2>&1 | grep ms/mode
python tools/als_sweep.py lbnl 16 f64 "" "slice_fill=0" 2>&1 | grep ms/iter
done > gpurun_out/s20_ab.log 2>&1
python tools/opt_sweep.py nell2 16 f64 "" "slice_fill=0" >> gpurun_out/s20_ab.log 2>&1
