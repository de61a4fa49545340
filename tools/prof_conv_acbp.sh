#!/bin/bash
# ncu --set full of the conv ACBP (im2col-mode TMA transform) at the ResNet-18
# CIFAR 64-channel shape (256 x 32 x 32 x 64, 3x3, stride 1).  TAG=x bash tools/prof_conv_acbp.sh
set -u
OUT=gpurun_out/prof_${TAG:-cacbp}
mkdir -p $OUT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 2 -c 1 \
  -o $OUT/cacbp python -c "
import sys, torch; sys.path.insert(0, '.')
from paper_2406_15102_b200 import ops
x = torch.randn(256, 32, 32, 64, device='cuda').to(torch.bfloat16)
for _ in range(3): ops.conv_acbp(x, 3, 1, 1, 0x5555, 8)
torch.cuda.synchronize()" > $OUT/ncu.log 2>&1
ncu -i $OUT/cacbp.ncu-rep --page raw --csv > $OUT/raw.csv 2>/dev/null
ncu -i $OUT/cacbp.ncu-rep --page source --csv --print-source sass > $OUT/sass.csv 2>/dev/null
gzip -f $OUT/raw.csv $OUT/sass.csv
rm -f $OUT/cacbp.ncu-rep
python tools/sass_summary.py $OUT/sass.csv.gz > $OUT/summary.md
