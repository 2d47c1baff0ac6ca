o=gpurun_out/s60_race.log; : > $o
run() { env "$@" timeout 300 python tools/race_hunt.py lbnl ${K:-10} 20 2>&1 | grep -v "odd traj\|rep " >> $o; }
K=10 run SPTK_DEFERRED_NORM=0
K=4 run SPTK_DEFERRED_NORM=0
K=4 run SPTK_X=0
K=1 run SPTK_X=0
K=1 run SPTK_DEFERRED_NORM=0
K=10 run SPTK_GAMMA_INV_CHOL=1
K=10 run RH_DET=1
K=10 run RH_DET=1 SPTK_DEFERRED_NORM=0
