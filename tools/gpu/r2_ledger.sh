python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/lg_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "perm or copies or shard or host or chunked or duplicate" > gpurun_out/lg_tests.log 2>&1
for k in 1 2 3; do python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e; done > gpurun_out/lg_bench3.jsonl 2> gpurun_out/lg_bench3.err
SPTK_NO_GRAPH=1 python tools/perm_timing.py nell2 1 > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:radix_ -s 20 -c 4 -o gpurun_out/radix python tools/perm_timing.py nell2 1 > gpurun_out/lg_ncu.log 2>&1
