for r in 1 2 3 4 5 6; do python bench.py --config lbnl --rank 16 --no-e2e --no-cpu-baseline > gpurun_out/s47_lbnl_$r.json 2> gpurun_out/s47_lbnl_$r.err; echo "lbnl $r rc=$?" >> gpurun_out/s47_rc.log; done
for r in 1 2 3; do python bench.py --config tiny --rank 8 --steps 20 --warmup 500 > gpurun_out/s47_tiny_$r.json 2> gpurun_out/s47_tiny_$r.err; echo "tiny $r rc=$?" >> gpurun_out/s47_rc.log; done
for r in 1 2 3; do python bench.py > gpurun_out/s47_nell2_$r.json 2> gpurun_out/s47_nell2_$r.err; echo "nell2 $r rc=$?" >> gpurun_out/s47_rc.log; done
