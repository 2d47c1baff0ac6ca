python -m pytest tests -m gpu -q > gpurun_out/s70_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s70_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s70_smoke.log
python bench.py > gpurun_out/s70_default.json 2> gpurun_out/s70_default.err
python bench.py --config lbnl --rank 16 > gpurun_out/s70_lbnl.json 2> gpurun_out/s70_lbnl.err
