for L in paper_1809_09175_b200/libsptk.so tools/abx/libS3.so tools/abx/libI8M4.so; do
  echo "== $L"
  SPTK_LIB=$L python tools/sort_ab.py nell2 "" "sort_v1=1" 2>&1 | grep -i "ms/mode\|error"
  SPTK_LIB=$L python tools/sort_ab.py lbnl "" "sort_v1=1" 2>&1 | grep -i "ms/mode\|error"
done > gpurun_out/s4_sortab.log 2>&1
