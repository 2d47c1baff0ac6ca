python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/ts_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/ceilings tools/ceilings.cu -lcuda >> gpurun_out/ts_build.log 2>&1
./tools/ceilings > gpurun_out/ceilings2.json 2> gpurun_out/ceilings2.log
timeout 900 python -m pytest tests/test_gpu.py -x -q -s -k "sharded or one_rank" > gpurun_out/ts_sharded.log 2>&1
timeout 300 python -m pytest tests/test_gpu_multirank.py -q -rs > gpurun_out/ts_multirank.log 2>&1
SPTK_NO_GRAPH=0 python tools/als_probe.py lbnl 16 6 > gpurun_out/ts_lbnl_probe.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ts_lbnl_launches.csv python tools/als_probe.py lbnl 16 6 > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ts_tiny_launches.csv python tools/als_probe.py tiny 8 6 > /dev/null 2>&1
python bench.py --config lbnl --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ts_bench_lbnl.json 2>&1
python bench.py --config tiny --rank 8 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ts_bench_tiny.json 2>&1
