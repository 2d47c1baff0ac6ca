python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s36_smoke.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/s36_tests.log 2>&1
python bench.py > gpurun_out/s36_default.json 2> gpurun_out/s36_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/s36_ref.json 2>&1
