SPTK_DEBUG_SETUP=1 python tools/first_build.py nell2 3 > gpurun_out/s18_first_build_a.log 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s18_bench_a.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s18_bench_b.json 2>&1
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s18_bench_c.json 2>&1
./tools/ceilings > gpurun_out/s18_ceilings.json 2> gpurun_out/s18_ceilings.log
