python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/fb_build.log 2>&1
for k in 1 2 3; do python tools/first_build.py nell2 1; done > gpurun_out/fb_lazy.log 2>&1
for k in 1 2 3; do CUDA_MODULE_LOADING=EAGER python tools/first_build.py nell2 1; done > gpurun_out/fb_eager.log 2>&1
python tools/first_build.py nell2 3 > gpurun_out/fb_same.log 2>&1
python tools/als_sweep.py tiny 8 f64 "" "run=16" "run=4" > gpurun_out/fb_tiny.log 2>&1
