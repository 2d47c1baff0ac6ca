./tools/ceilings > gpurun_out/s30_ceilings.json 2> gpurun_out/s30_ceilings.log
cp gpurun_out/s30_ceilings.json profiles/ceilings.json
python bench.py --dtype f32 --no-cpu-baseline --no-e2e > gpurun_out/s30_f32.json 2> gpurun_out/s30_f32.err
python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s30_f64.json 2> gpurun_out/s30_f64.err
