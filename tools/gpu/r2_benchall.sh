python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/ba_build.log 2>&1
python bench.py > gpurun_out/ba_default.json 2> gpurun_out/ba_default.err
bash tools/bench_all.sh gpurun_out/ba_all.jsonl
SPTK_FORCE_SHARDED=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ba_sharded.json 2> gpurun_out/ba_sharded.err
python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/ba_single.json 2>&1
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ba_ref.json 2>&1
