python -c "import __graft_entry__ as g; g.build()" > gpurun_out/h_build.log 2>&1
python tools/opt_sweep.py delicious 16 f64 "hot_l2_kb=0" "" "hot_l2_kb=32768" "hot_l2_kb=98304" "hot_l2_kb=16384" > gpurun_out/h_del.log 2>&1
python tools/opt_sweep.py nell2 16 f64 "hot_l2_kb=0" "" > gpurun_out/h_nell.log 2>&1
python tools/opt_sweep.py amazon 16 f64 "hot_l2_kb=0" "" > gpurun_out/h_amz.log 2>&1
python tools/opt_sweep.py lbnl 16 f64 "hot_l2_kb=0" "" > gpurun_out/h_lbnl.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q -k "delicious or lbnl" > gpurun_out/h_exact.log 2>&1
