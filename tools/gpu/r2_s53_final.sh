python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s53_smoke.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s53_tests.log 2>&1
