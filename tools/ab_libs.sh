#!/bin/bash
# A/B timing of two builds of libtagdsp_gpu.so on one box, alternated so that
# both see the same thermal / power-cap state: copy the builds to
# abtest/lib_A.so and abtest/lib_B.so (git-ignored, they travel with gpurun),
# then: gpurun -- 'bash tools/ab_libs.sh gpurun_out/ab'
OUT=${1:-gpurun_out/ab}; mkdir -p "$OUT"
python tools/sweep.py "" "" "" "" > /dev/null 2>&1   # warm the GPU
for i in 1 2 3 4; do
  for v in A B; do
    TDG_LIB_PATH=abtest/lib_$v.so python tools/sweep.py "" "" "" | tail -2 | sed "s/^/$v /" >> "$OUT/ab.txt"
  done
done
