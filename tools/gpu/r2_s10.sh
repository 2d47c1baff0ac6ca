timeout 900 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded" > gpurun_out/s10_tests.log 2>&1
for cfg in "lbnl 16 f64" "delicious 16 f64" "tiny 8 f64"; do
  python tools/als_sweep.py $cfg "" "apply_mma=0" 2>&1 | grep ms/iter
done > gpurun_out/s10_ab.log 2>&1
ncu --set full --cache-control none --clock-control none -k regex:apply_gram_mma -s 4 -c 1 -o gpurun_out/s10_apply_mma python tools/als_probe.py lbnl 16 3 > gpurun_out/s10_ncu.log 2>&1
ncu -i gpurun_out/s10_apply_mma.ncu-rep --page raw --csv > gpurun_out/s10_apply_mma_raw.csv 2>/dev/null
python tools/timeline.py tiny 8 20 > gpurun_out/s10_tl_tiny.log 2>&1
python tools/timeline.py lbnl 16 10 > gpurun_out/s10_tl_lbnl.log 2>&1
