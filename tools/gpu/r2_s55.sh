for r in 1 2 3 4 5; do python bench.py --config lbnl --rank 16 --steps 20 > gpurun_out/s55_lbnl_$r.json 2> gpurun_out/s55_lbnl_$r.err; echo "lbnl $r rc=$?" >> gpurun_out/s55_rc.log; done
