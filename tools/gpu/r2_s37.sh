timeout 900 python -m pytest tests/test_gpu.py -x -q -k "slice_traversal" -rs > gpurun_out/s37_tests.log 2>&1
for r in 1 2; do
python tools/opt_sweep.py nell2 16 f64 "" "slice_smem=64" "slice_smem=48" "slice_smem=96" 2>&1 | grep ms/mode
done > gpurun_out/s37_ab.log 2>&1
python tools/opt_sweep.py nell2 16 f32 "" "slice_smem=64" "slice_smem=32" >> gpurun_out/s37_ab.log 2>&1
python tools/opt_sweep.py lbnl 16 f64 "" "slice_smem=64" >> gpurun_out/s37_ab.log 2>&1
