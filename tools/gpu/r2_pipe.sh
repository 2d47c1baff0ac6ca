python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/pp_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_exact.py -x -q -k "pipe and (tiny or lbnl or nell2 or delicious)" > gpurun_out/pp_exact.log 2>&1
for L in paper_1809_09175_b200/libsptk.so tools/abx/libD3.so tools/abx/libD6.so; do
  echo "== $L"
  SPTK_LIB=$L python tools/opt_sweep.py delicious 16 f64 "" "variant=3" "variant=3,rowrec=0" 2>&1 | grep ms/mode
  SPTK_LIB=$L python tools/opt_sweep.py amazon 16 f64 "" "slice=0,variant=3" "slice=0" 2>&1 | grep ms/mode
done > gpurun_out/pp_ab.log 2>&1
python tools/opt_sweep.py nell2 16 f64 "" "slice=0,variant=3" "slice=0" >> gpurun_out/pp_ab.log 2>&1
python tools/opt_sweep.py lbnl 16 f64 "" "slice=0,variant=3" >> gpurun_out/pp_ab.log 2>&1
