python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/g3_build.log 2>&1
timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/g3_tests.log 2>&1
for cfg in "lbnl 16 f64" "delicious 16 f64"; do
  for L in tools/abx/libbase.so paper_1809_09175_b200/libsptk.so; do
    echo "== $L $cfg"; SPTK_LIB=$L python tools/als_sweep.py $cfg "" 2>&1 | grep ms/iter
  done
done > gpurun_out/g3_ab.log 2>&1
python tools/als_sweep.py tiny 8 f64 "" "small_iter=0" >> gpurun_out/g3_ab.log 2>&1
