python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/cs_build.log 2>&1
python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/cs_ab.log 2>&1
SPTK_COPY_SEC=1,2,1,1 python tools/opt_sweep.py delicious 16 f64 "" >> gpurun_out/cs_ab.log 2>&1
SPTK_COPY_SEC=1,2,1,2 python tools/opt_sweep.py delicious 16 f64 "" >> gpurun_out/cs_ab.log 2>&1
SPTK_COPY_SEC=-1,-1,-1,-1 python tools/opt_sweep.py delicious 16 f64 "" >> gpurun_out/cs_ab.log 2>&1
