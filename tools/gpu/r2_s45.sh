for r in 1 2; do python bench.py --config tiny --rank 8 --steps 20 --warmup 500 --no-e2e --no-cpu-baseline > gpurun_out/s45_tiny_$r.json 2>/dev/null; done
for r in 1 2; do python bench.py --config lbnl --rank 16 --no-e2e --no-cpu-baseline > gpurun_out/s45_lbnl_$r.json 2>/dev/null; done
