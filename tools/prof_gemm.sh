#!/bin/bash
# ncu --set full of the fc2 dX GEMM (25216 x 3072 x 768, bf16 out) in the
# single-CTA (BN 256) and CTA-pair (BN 256) variants.  TAG=x bash tools/prof_gemm.sh
set -u
TAG=${TAG:-gemm}
OUT=gpurun_out/prof_${TAG}
mkdir -p $OUT
for v in c p; do
  if [ $v = c ]; then export HLQ_GEMM_PAIR=0; else export HLQ_GEMM_PAIR=1; fi
  HLQ_GEMM_BN=256 timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 2 -c 1 \
    -o $OUT/fc2dx_$v python tools/gemm_one.py 25216,3072,768 int8 > $OUT/$v.log 2>&1
  ncu -i $OUT/fc2dx_$v.ncu-rep --page raw --csv > $OUT/fc2dx_${v}_raw.csv 2>/dev/null
  ncu -i $OUT/fc2dx_$v.ncu-rep --page source --csv --print-source sass > $OUT/fc2dx_${v}_sass.csv 2>/dev/null
  gzip -f $OUT/fc2dx_${v}_raw.csv $OUT/fc2dx_${v}_sass.csv
  rm -f $OUT/fc2dx_$v.ncu-rep
done
ls -la $OUT
