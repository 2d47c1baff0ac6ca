python tools/repro_singular.py lbnl 16 12 "" "gj_warp=0" "side_prio=0" "fused_reduce=0" "apply_mma=0" "prezero=0" > gpurun_out/s48_repro.log 2>&1
