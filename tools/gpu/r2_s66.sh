python -m pytest tests -m gpu -q > gpurun_out/s66_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s66_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s66_smoke.log
python bench.py > gpurun_out/s66_default.json 2> gpurun_out/s66_default.err
python bench.py --config lbnl --rank 16 > gpurun_out/s66_lbnl.json 2> gpurun_out/s66_lbnl.err
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s66_ref.json 2> gpurun_out/s66_ref.err
