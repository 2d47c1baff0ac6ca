for r in 1 2 3 4; do python bench.py --config lbnl --rank 16 --no-e2e --no-cpu-baseline > gpurun_out/s46_lbnl_$r.json 2> gpurun_out/s46_lbnl_$r.err; echo "rc=$?" >> gpurun_out/s46_rc.log; done
