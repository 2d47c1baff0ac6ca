for r in 1 2; do
PYTORCH_NO_CUDA_MEMORY_CACHING=1 python tools/alloc_probe.py 0 >> gpurun_out/s38_alloc.log 2>&1
PYTORCH_NO_CUDA_MEMORY_CACHING=1 python tools/alloc_probe.py 12 >> gpurun_out/s38_alloc.log 2>&1
done
