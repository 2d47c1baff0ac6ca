#!/bin/bash
# One bench line per BASELINE config (1 GPU) -> $1 (jsonl).  Usage: tools/bench_all.sh out.jsonl
out=${1:-gpurun_out/bench_all.jsonl}
: > "$out"
run() { python bench.py "$@" 2>>"${out%.jsonl}.err" | tail -1 >> "$out"; }
run --config tiny --rank 8 --steps 20 --warmup 500 --no-e2e
run --config lbnl --rank 16
run --config nell2 --rank 16 --dtype f64
run --config nell2 --rank 64 --dtype f64 --no-cpu-baseline
run --config nell2 --rank 16 --dtype f32 --no-cpu-baseline
run --config nell2 --rank 64 --dtype f32 --no-cpu-baseline
run --config nell2 --rank 16 --dtype f64 --layout perm_gather --no-cpu-baseline --no-e2e
run --config nell2 --rank 17 --dtype f64 --no-cpu-baseline --no-e2e
run --config delicious --rank 16 --steps 20
run --config amazon --rank 16 --steps 10
