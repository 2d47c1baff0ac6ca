python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/pd_build.log 2>&1
python tools/als_sweep.py tiny 8 f64 "pdl=0" "" "run=4" "run=8" "run=4,pdl=0" > gpurun_out/pd_ab.log 2>&1
python tools/als_sweep.py lbnl 16 f64 "pdl=0" "" >> gpurun_out/pd_ab.log 2>&1
python tools/als_sweep.py nell2 16 f64 "pdl=0" "" >> gpurun_out/pd_ab.log 2>&1
python tools/als_sweep.py delicious 16 f64 "pdl=0" "" >> gpurun_out/pd_ab.log 2>&1
timeout 2400 python -m pytest tests/ -x -q -m gpu > gpurun_out/pd_tests.log 2>&1
