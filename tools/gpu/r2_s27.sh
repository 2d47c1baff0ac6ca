python tools/opt_sweep.py lbnl 16 f64 "" "run=16" "run=32" "run=64" "run=128" "rowrec=0" "variant=1" > gpurun_out/s27_tall.log 2>&1
