python -c "import __graft_entry__ as g; g.build()" > gpurun_out/r2x_build.log 2>&1
timeout 2400 python -m pytest tests/test_gpu_exact.py -x -q -s -rs --durations=15 > gpurun_out/r2x_exact.log 2>&1
timeout 1200 python -m pytest tests/test_gpu.py -x -q -s -k "config or ridge" --durations=10 > gpurun_out/r2x_full.log 2>&1
