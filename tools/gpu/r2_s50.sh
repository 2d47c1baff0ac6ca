python tools/repro_singular2.py lbnl > gpurun_out/s50_repro2.log 2>&1
