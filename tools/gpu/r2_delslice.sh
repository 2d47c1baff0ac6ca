python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/ds_build.log 2>&1
python tools/opt_sweep.py delicious 16 f64 "" "slice=2" "slice=2,slice_l2_kb=65536" "slice=2,slice_l2_kb=131072" > gpurun_out/ds_ab.log 2>&1
SPTK_COPY_SEC=2,0,0,1 python tools/opt_sweep.py delicious 16 f64 "" "slice=2" "slice=2,slice_l2_kb=65536" "slice=2,slice_l2_kb=131072" "slice=2,slice_l2_kb=262144" >> gpurun_out/ds_ab.log 2>&1
SPTK_COPY_SEC=1,0,1,1 python tools/opt_sweep.py delicious 16 f64 "" "slice=2" "slice=2,slice_l2_kb=131072" >> gpurun_out/ds_ab.log 2>&1
