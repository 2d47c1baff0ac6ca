python -m pytest tests -m gpu -q > gpurun_out/s63_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s63_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/s63_smoke.log
bash tools/bench_all.sh gpurun_out/s63_all.jsonl
python bench.py > gpurun_out/s63_default.json 2> gpurun_out/s63_default.err
