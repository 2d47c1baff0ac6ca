timeout 900 python -m pytest tests/test_gpu.py -x -q -k "window_major" > gpurun_out/s16_tests.log 2>&1
REPS=1 ncu --set full --clock-control none -k regex:mttkrp_coop -s 23 -c 1 -o gpurun_out/s16_nowin python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s16_ncu0.log 2>&1
REPS=1 SPTK_WIN=1 ncu --set full --clock-control none -k regex:mttkrp_coop -s 23 -c 1 -o gpurun_out/s16_win python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s16_ncu1.log 2>&1
for f in s16_nowin s16_win; do ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv 2>/dev/null; done
