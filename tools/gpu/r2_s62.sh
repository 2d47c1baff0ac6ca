python -m pytest tests -m gpu -x -q -k "cp_als" > gpurun_out/s62_tests.log 2>&1
o=gpurun_out/s62_race.log; : > $o
run() { env "$@" timeout 300 python tools/race_hunt.py lbnl ${K:-10} 40 2>&1 | grep -v "odd traj" >> $o; }
run SPTK_X=0
run SPTK_NO_GRAPH=1
K=30 run SPTK_X=0
timeout 600 python tools/defer_vs_explicit.py lbnl 10 > gpurun_out/s62_dve.log 2>&1
