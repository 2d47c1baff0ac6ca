#!/bin/bash
# Slice traversal A/B and slice-length sweep on the NELL-2 shape (GPU box).
# Usage: tools/slice_sweep.sh > gpurun_out/sweep_slice.log
for rows in 1024 2048 4096; do
  for c in "nell2 16 f64" "nell2 16 f32"; do
    echo "== SPTK_SLICE_ROWS=$rows $c"
    SPTK_SLICE_ROWS=$rows VARIANTS=-2 RUNS=-2 python tools/sweep.py $c 2>&1 | tail -1
  done
done
for R in 8 16 32 64 128; do
  for dt in f64 f32; do
    for o in 0 1; do
      echo "== SPTK_SLICE=$o nell2 $R $dt"
      SPTK_SLICE=$o VARIANTS=-2 RUNS=-2 python tools/sweep.py nell2 $R $dt 2>&1 | tail -1
    done
  done
done
