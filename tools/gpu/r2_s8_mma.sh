timeout 1500 python -m pytest tests/test_gpu.py -x -q -k "cp_als or sharded or config" > gpurun_out/s8_tests.log 2>&1
for cfg in "lbnl 16 f64" "delicious 16 f64" "nell2 16 f64" "tiny 8 f64" "nell2 16 f32"; do
  python tools/als_sweep.py $cfg "" "apply_mma=0" "apply_mma=0,prezero=0" 2>&1 | grep ms/iter
done > gpurun_out/s8_ab.log 2>&1
ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/s8_lbnl_launches.csv python tools/als_probe.py lbnl 16 8 > gpurun_out/s8_lbnl_probe.log 2>&1
ncu --set full --cache-control none --clock-control none -k regex:apply_gram_mma -s 30 -c 1 -o gpurun_out/s8_apply_mma python tools/als_probe.py lbnl 16 8 > gpurun_out/s8_ncu.log 2>&1
ncu -i gpurun_out/s8_apply_mma.ncu-rep --page raw --csv > gpurun_out/s8_apply_mma_raw.csv 2>/dev/null
