for r in 1 2; do
python tools/opt_sweep.py nell2 16 f64 "" > gpurun_out/s25_def_$r.log 2>&1
SPTK_COPY_SEC=1,0,0 python tools/opt_sweep.py nell2 16 f64 "" > gpurun_out/s25_sec100_$r.log 2>&1
SPTK_COPY_SEC=2,2,1 python tools/opt_sweep.py nell2 16 f64 "" > gpurun_out/s25_sec221_$r.log 2>&1
done
python tools/opt_sweep.py nell2 16 f64 "" "slice_rows=2048" "slice_rows=8192" > gpurun_out/s25_rows.log 2>&1
