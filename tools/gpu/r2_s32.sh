timeout 1500 python -m pytest tests/test_gpu.py -x -q -k "perm or copy or cp_als_full_size or build" > gpurun_out/s32_tests.log 2>&1
for r in 1 2 3; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s32_bench_$r.json 2>/dev/null; done
python bench.py --config delicious --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s32_bench_del.json 2>/dev/null
