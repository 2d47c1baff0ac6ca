python bench.py --config tiny --rank 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/st_tiny20.json 2>&1
python bench.py --config tiny --rank 8 --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/st_tiny200.json 2>&1
python bench.py --config lbnl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/st_lbnl20.json 2>&1
python bench.py --config lbnl --steps 200 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/st_lbnl200.json 2>&1
python tools/opt_sweep.py lbnl 16 f64 "" "slice_rows=2048" "slice_rows=1024" "slice_rows=512" > gpurun_out/st_lbnl_slice.log 2>&1
python tools/opt_sweep.py nell2 16 f64 "" "slice_rows=2048" > gpurun_out/st_nell_slice.log 2>&1
