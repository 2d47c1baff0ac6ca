o=gpurun_out/s58_race.log; : > $o
run() { env "$@" timeout 300 python tools/race_hunt.py lbnl 10 40 2>&1 | grep -v "rep " >> $o; }
run SPTK_X=0
run SPTK_TAIL_ROWS=0
run SPTK_APPLY_WARP=0 SPTK_APPLY_MMA=0
run SPTK_GENERIC=1
run SPTK_SLICE=0
run SPTK_VARIANT=0
run SPTK_VARIANT=1
run SPTK_USE_COPY=0
run SPTK_SIDE_PRIO=0
run SPTK_ROWREC=0
run SPTK_RUN=64
