python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/w_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/w_tests.log 2>&1
python tools/als_sweep.py lbnl 16 f64 "apply_warp=0" "" > gpurun_out/w_ab.log 2>&1
python tools/als_sweep.py tiny 8 f64 "apply_warp=0" "" >> gpurun_out/w_ab.log 2>&1
python tools/als_sweep.py nell2 16 f64 "apply_warp=0" "" >> gpurun_out/w_ab.log 2>&1
python tools/als_sweep.py delicious 16 f64 "apply_warp=0" "" >> gpurun_out/w_ab.log 2>&1
python tools/als_sweep.py nell2 16 f32 "apply_warp=0" "" >> gpurun_out/w_ab.log 2>&1
python tools/als_sweep.py paper_synth 32 f64 "apply_warp=0" "" >> gpurun_out/w_ab.log 2>&1
