timeout 900 python -m pytest tests/test_gpu.py -x -q -k "degenerate or cp_als_full_size or tiny_trajectory" -rs > gpurun_out/s51_tests.log 2>&1
for r in 1 2 3 4 5 6; do python bench.py --config lbnl --rank 16 --no-cpu-baseline > gpurun_out/s51_lbnl_$r.json 2> gpurun_out/s51_lbnl_$r.err; echo "lbnl $r rc=$?" >> gpurun_out/s51_rc.log; done
python bench.py > gpurun_out/s51_nell2.json 2> gpurun_out/s51_nell2.err; echo "nell2 rc=$?" >> gpurun_out/s51_rc.log
python tools/repro_singular2.py lbnl > gpurun_out/s51_repro2.log 2>&1
