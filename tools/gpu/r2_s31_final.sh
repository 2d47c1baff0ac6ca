python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s31_smoke.log 2>&1
python bench.py > gpurun_out/s31_default1.json 2> gpurun_out/s31_default1.err
python bench.py > gpurun_out/s31_default2.json 2> gpurun_out/s31_default2.err
bash tools/bench_all.sh gpurun_out/s31_all.jsonl
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s31_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s31_ncu_bench.log 2>&1
