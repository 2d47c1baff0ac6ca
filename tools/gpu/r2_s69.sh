python -m pytest tests -m gpu -q -x -k "prezero or cp_als_full_size or smoke" > gpurun_out/s69_tests.log 2>&1
REPS=5 ITERS=50 timeout 600 python tools/als_sweep.py lbnl 16 f64 "" "prezero_mb=64,zero_in_apply=1" "" "prezero_mb=64,zero_in_apply=1" > gpurun_out/s69_ab.log 2>&1
REPS=3 ITERS=10 timeout 900 python tools/als_sweep.py delicious 16 f64 "" "zero_in_apply=1" "" "zero_in_apply=1" >> gpurun_out/s69_ab.log 2>&1
SPTK_PREZERO_MB=64 SPTK_ZERO_IN_APPLY=1 timeout 300 python tools/race_hunt.py lbnl 10 20 2>&1 | grep -v "odd traj" >> gpurun_out/s69_ab.log
timeout 300 python tools/race_hunt.py lbnl 10 20 2>&1 | grep -v "odd traj" >> gpurun_out/s69_ab.log
python tools/timeline.py lbnl 16 10 f64 prezero_mb=64,zero_in_apply=1 > gpurun_out/s69_tl_lbnl.log 2>&1
