#!/bin/bash
# Round-2 ncu captures of the dominant kernel (the fused dual gy transform at the
# ViT-B/16 fc1 shape, as the training path runs it: with the column sums).
# Usage (under gpurun, one GPU):  ROUND=r02 TAG=base bash tools/prof_r02.sh
set -u
TAG=${TAG:-base}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 4 -c 1 \
  -o $OUT/dual python tools/prof_driver.py dualcs 128,197,768,3072 2 > $OUT/ncu.log 2>&1
ncu -i $OUT/dual.ncu-rep --page source --csv --print-source sass > $OUT/dual_sass.csv 2>/dev/null
ncu -i $OUT/dual.ncu-rep --page raw --csv > $OUT/dual_raw.csv 2>/dev/null
gzip -f $OUT/dual_sass.csv $OUT/dual_raw.csv
rm -f $OUT/dual.ncu-rep
ls -la $OUT
