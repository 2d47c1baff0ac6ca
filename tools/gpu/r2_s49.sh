SPTK_LIB=tools/abx/libstart.so python tools/repro_singular.py lbnl 16 16 "" > gpurun_out/s49_repro.log 2>&1
python tools/repro_singular.py lbnl 16 16 "" "pdl=0" >> gpurun_out/s49_repro.log 2>&1
