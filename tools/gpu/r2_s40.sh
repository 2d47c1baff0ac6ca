for r in 1 2 3; do
python -c "import __graft_entry__ as g; g.smoke()" > /dev/null 2>&1
sleep 3
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/s40_bench_$r.json 2>/dev/null
done
