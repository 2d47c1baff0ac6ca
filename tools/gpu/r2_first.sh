set -x
nproc; free -g; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2_smoke.log 2>&1
python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2_bench0.json 2> gpurun_out/r2_bench0.err
python bench.py --config delicious --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_del.json 2> gpurun_out/r2_bench_del.err
python bench.py --config lbnl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_lbnl.json 2>&1
python bench.py --config tiny --rank 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/r2_bench_tiny.json 2>&1
