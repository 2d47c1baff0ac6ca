timeout 900 python -m pytest tests/test_gpu.py -x -q -k "window_major or perm_bitexact" > gpurun_out/s15_tests.log 2>&1
for r in 1 2; do
python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s15_win0_$r.log 2>&1
SPTK_WIN=1 python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s15_win1_$r.log 2>&1
SPTK_WIN=1 SPTK_SLICE_L2_KB=16384 python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s15_win1_16m_$r.log 2>&1
done
SPTK_WIN=1 ncu --set full --clock-control none -k regex:mttkrp_coop -s 1 -c 1 -o gpurun_out/s15_win python tools/opt_sweep.py delicious 16 f64 "" > gpurun_out/s15_ncu.log 2>&1
ncu -i gpurun_out/s15_win.ncu-rep --page raw --csv > gpurun_out/s15_win_raw.csv 2>/dev/null
