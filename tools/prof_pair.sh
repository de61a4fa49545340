#!/bin/bash
# ncu --set full of the fused dW + dX CTA-pair launch at the ViT fc2 shape.
set -u
OUT=gpurun_out/prof_${TAG:-pair}
mkdir -p $OUT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_i8_2sm -s 1 -c 1 \
  -o $OUT/fc2pair python tools/prof_driver.py gemm_pair 128,197,3072,768 2 > $OUT/ncu.log 2>&1
ncu -i $OUT/fc2pair.ncu-rep --page raw --csv > $OUT/fc2pair_raw.csv 2>/dev/null
ncu -i $OUT/fc2pair.ncu-rep --page source --csv --print-source sass > $OUT/fc2pair_sass.csv 2>/dev/null
gzip -f $OUT/fc2pair_raw.csv $OUT/fc2pair_sass.csv
rm -f $OUT/fc2pair.ncu-rep
