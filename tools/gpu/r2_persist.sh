python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ps_build.log 2>&1
python tools/opt_sweep.py delicious 16 f64 "hot_l2_kb=0" "hot_l2_kb=65536" "hot_l2_kb=0,l2_persist_kb=-1" "hot_l2_kb=65536,l2_persist_kb=-1" "hot_l2_kb=98304,l2_persist_kb=-1" "hot_l2_kb=32768,l2_persist_kb=-1" "hot_l2_kb=0,l2_persist_kb=0" > gpurun_out/ps_del.log 2>&1
