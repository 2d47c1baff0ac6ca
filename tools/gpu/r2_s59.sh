o=gpurun_out/s59_race.log; : > $o
run() { env "$@" timeout 300 python tools/race_hunt.py lbnl ${K:-10} 40 >> $o 2>&1; }
run SPTK_X=0
run SPTK_NO_GRAPH=1
K=4 run SPTK_X=0
