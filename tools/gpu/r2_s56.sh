for r in 1 2 3 4 5 6 7 8; do python bench.py --config lbnl --rank 16 --steps 10 > gpurun_out/s56_lbnl_$r.json 2> gpurun_out/s56_lbnl_$r.err; echo "lbnl10 $r rc=$?" >> gpurun_out/s56_rc.log; done
