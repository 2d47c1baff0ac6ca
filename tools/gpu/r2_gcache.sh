timeout 1200 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded or tiny or host or chunked" > gpurun_out/gc_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/gc_tests.log 2>&1
python bench.py --config tiny --rank 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gc_tiny20.json 2>&1
python bench.py --config tiny --rank 8 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/gc_tiny50.json 2>&1
python bench.py --config lbnl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/gc_lbnl20.json 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/gc_nell20.json 2>&1
