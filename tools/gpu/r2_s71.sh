python bench.py > gpurun_out/s71_default.json 2> gpurun_out/s71_default.err
python bench.py --config lbnl --rank 16 > gpurun_out/s71_lbnl.json 2> gpurun_out/s71_lbnl.err
python bench.py --config tiny --rank 8 --no-e2e > gpurun_out/s71_tiny.json 2> gpurun_out/s71_tiny.err
