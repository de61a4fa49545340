#!/bin/bash
# ncu --set full of the fused dual transform's two passes launched alone (fc1
# gy shape), SASS source pages summarised (tools/sass_summary.py).
# Usage (under gpurun, one GPU):  TAG=x bash tools/prof_passes.sh
set -u
TAG=${TAG:-passes}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
for what in statspass quantpass; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 4 -c 1 \
    -o $OUT/$what python tools/prof_driver.py $what 128,197,768,3072 3 > $OUT/$what.log 2>&1
  ncu -i $OUT/$what.ncu-rep --page source --csv --print-source sass > $OUT/${what}_sass.csv 2>/dev/null
  ncu -i $OUT/$what.ncu-rep --page raw --csv > $OUT/${what}_raw.csv 2>/dev/null
  gzip -f $OUT/${what}_sass.csv $OUT/${what}_raw.csv
  rm -f $OUT/$what.ncu-rep
done
python tools/sass_summary.py $OUT/statspass_sass.csv.gz $OUT/quantpass_sass.csv.gz > $OUT/summary.md
ls -la $OUT
