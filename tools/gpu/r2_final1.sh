python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f1_smoke.log 2>&1
timeout 3000 python -m pytest tests/ -x -q -m gpu -rs > gpurun_out/f1_tests.log 2>&1
bash tools/bench_all.sh gpurun_out/f1_all.jsonl
python bench.py > gpurun_out/f1_default.json 2> gpurun_out/f1_default.err
python bench.py > gpurun_out/f1_default2.json 2> gpurun_out/f1_default2.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/f1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/f1_ncu_bench.log 2>&1
