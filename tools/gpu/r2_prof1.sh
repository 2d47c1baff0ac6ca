set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p1_build.log 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/ceilings tools/ceilings.cu
./tools/ceilings > gpurun_out/ceilings.json 2> gpurun_out/ceilings.log
# Delicious: plain run first, then one full capture of the 4 MTTKRP launches of an iteration
SPTK_NO_GRAPH=1 python tools/als_probe.py delicious 16 1 > gpurun_out/p1_del.log 2>&1 && \
SPTK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:mttkrp_ -c 4 \
   -o gpurun_out/del_mttkrp python tools/als_probe.py delicious 16 1 > gpurun_out/p1_del_ncu.log 2>&1
SPTK_NO_GRAPH=1 python tools/als_probe.py nell2 16 1 > gpurun_out/p1_nell.log 2>&1 && \
SPTK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:mttkrp_ -c 3 \
   -o gpurun_out/nell2_mttkrp python tools/als_probe.py nell2 16 1 > gpurun_out/p1_nell_ncu.log 2>&1
bash tools/traffic_capture.sh > gpurun_out/p1_traffic.log 2>&1
