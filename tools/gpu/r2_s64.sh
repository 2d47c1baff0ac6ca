python -m pytest tests -m gpu -q > gpurun_out/s64_tests.log 2>&1
REPS=5 ITERS=50 timeout 900 python tools/als_sweep.py lbnl 16 f64 "" "tail_rows=0" "tail_rows=2000" "apply_tile=32" "apply_tile=128" "apply_nb_mult=2" "slice_fill=4" "slice_fill=10" "side_prio=0" "fused_reduce=0" "apply_wave=0" > gpurun_out/s64_sweep.log 2>&1
