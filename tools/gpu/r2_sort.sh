python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/s_build.log 2>&1
for L in paper_1809_09175_b200/libsptk.so tools/abx/libmatch.so paper_1809_09175_b200/libsptk.so tools/abx/libmatch.so; do
  echo "== $L"; SPTK_LIB=$L python tools/perm_timing.py nell2 2 2>&1 | grep "pass 1 rep 1"
  SPTK_LIB=$L python tools/perm_timing.py delicious 2 2>&1 | grep "pass 1 rep 1"
done > gpurun_out/s_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu.py -x -q -k "perm" > gpurun_out/s_tests.log 2>&1
