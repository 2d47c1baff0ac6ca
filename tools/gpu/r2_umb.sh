python -c "import __graft_entry__ as g; g.build()" > gpurun_out/u_build.log 2>&1
for L in paper_1809_09175_b200/libsptk.so tools/abx/libU1M2.so tools/abx/libU1M3.so tools/abx/libU1M4.so paper_1809_09175_b200/libsptk.so; do
  echo "== $L"; SPTK_LIB=$L python tools/opt_sweep.py delicious 16 f64 "" 2>&1 | grep ms/mode
  SPTK_LIB=$L python tools/opt_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/mode
done > gpurun_out/u_ab.log 2>&1
