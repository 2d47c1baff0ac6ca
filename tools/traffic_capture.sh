#!/bin/bash
# ncu DRAM bytes + duration of the MTTKRP launches of one CP-ALS iteration per
# bench workload -> gpurun_out/traffic_<key>.csv (plain run first, as required).
# Usage (GPU box): tools/traffic_capture.sh
set -u
run() {  # key config R dtype [env]
  local key=$1 cfg=$2 R=$3 dt=$4 extra=${5:-}
  local B="python tools/als_probe.py $cfg $R 1 $dt"
  env $extra SPTK_NO_GRAPH=1 $B > gpurun_out/tp_$key.log 2>&1 && \
  env $extra SPTK_NO_GRAPH=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:mttkrp_ --csv --log-file gpurun_out/traffic_$key.csv $B > /dev/null 2>&1
  echo "$key rc=$?"
}
run nell2_R16_f64 nell2 16 f64
run nell2_R16_f64_perm_gather nell2 16 f64 SPTK_USE_COPY=0
run nell2_R64_f64 nell2 64 f64
run nell2_R16_f32 nell2 16 f32
run nell2_R64_f32 nell2 64 f32
run lbnl_R16_f64 lbnl 16 f64
run delicious_R16_f64 delicious 16 f64
run amazon_R16_f64 amazon 16 f64
run tiny_R8_f64 tiny 8 f64
