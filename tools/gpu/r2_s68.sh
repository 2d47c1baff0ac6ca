python -m pytest tests -m gpu -q > gpurun_out/s68_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s68_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s68_smoke.log
python bench.py > gpurun_out/s68_default.json 2> gpurun_out/s68_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s68_launches.csv python bench.py --steps 2 --warmup 3 > gpurun_out/s68_ncu.log 2>&1
