python tools/repro_singular2.py lbnl 10,20,30,40 > gpurun_out/s52_lbnl.log 2>&1
python tools/repro_singular2.py nell2 60,120 > gpurun_out/s52_nell2.log 2>&1
python tools/repro_singular2.py tiny 60,120,600 8 > gpurun_out/s52_tiny.log 2>&1
