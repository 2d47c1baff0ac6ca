o=gpurun_out/s57_race.log; : > $o
run() { env "$@" timeout 300 python tools/race_hunt.py lbnl 10 30 >> $o 2>&1; }
run SPTK_X=0
run SPTK_PDL=0
run SPTK_NO_GRAPH=1
run SPTK_FUSED_REDUCE=0
run SPTK_APPLY_MMA=0
run SPTK_GJ_WARP=0
run SPTK_DEFERRED_NORM=0
run SPTK_PREZERO=0
run SPTK_PDL=0 SPTK_NO_GRAPH=1 SPTK_FUSED_REDUCE=0 SPTK_APPLY_MMA=0 SPTK_GJ_WARP=0
