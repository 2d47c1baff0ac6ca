python -c "import paper_1809_09175_b200 as sp; print(sp.version())" > gpurun_out/g_build.log 2>&1
python tools/als_sweep.py lbnl 16 f64 "" "apply_tile=128" "apply_tile=256" "apply_nb_mult=2" "apply_nb_mult=4" "apply_wave=0" "tail_rows=8192" "apply_wave=0,apply_nb_mult=4" > gpurun_out/g_lbnl.log 2>&1
python tools/als_sweep.py tiny 8 f64 "" "apply_tile=16" "apply_tile=32" > gpurun_out/g_tiny.log 2>&1
SPTK_NO_GRAPH=1 python tools/als_probe.py lbnl 16 1 > /dev/null 2>&1 && SPTK_NO_GRAPH=1 ncu --set full --import-source on --clock-control none -k regex:apply_gram -s 4 -c 1 -o gpurun_out/lbnl_apply python tools/als_probe.py lbnl 16 1 > gpurun_out/g_ncu.log 2>&1
