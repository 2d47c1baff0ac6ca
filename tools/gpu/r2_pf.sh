python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/pf_build.log 2>&1
for L in paper_1809_09175_b200/libsptk.so tools/abx/libpf.so; do
  echo "== $L"; SPTK_LIB=$L python tools/opt_sweep.py delicious 16 f64 "" 2>&1 | grep ms/mode
  SPTK_LIB=$L python tools/opt_sweep.py amazon 16 f64 "" "slice=0" 2>&1 | grep ms/mode
  SPTK_LIB=$L python tools/opt_sweep.py lbnl 16 f64 "" 2>&1 | grep ms/mode
done > gpurun_out/pf_ab.log 2>&1
python tools/als_sweep.py tiny 8 f64 "" >> gpurun_out/pf_ab.log 2>&1
for k in 1 2 3; do python tools/first_build.py nell2 1; done > gpurun_out/pf_first.log 2>&1
SPTK_DEBUG_SETUP=1 python tools/first_build.py nell2 2 >> gpurun_out/pf_first.log 2>&1
python tools/perm_timing.py nell2 2 > gpurun_out/pf_perm.log 2>&1
