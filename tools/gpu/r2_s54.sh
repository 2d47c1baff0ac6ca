bash tools/bench_all.sh gpurun_out/s54_all.jsonl
