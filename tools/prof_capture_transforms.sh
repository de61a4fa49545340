#!/bin/bash
# Transform / conv ncu captures (their --set full reports are large: summarised
# on the box, only the summary comes back).  Run under gpurun from the repo root.
set -u
mkdir -p gpurun_out/tr
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 1 -c 1 \
  -o gpurun_out/tr/prof_dual python tools/prof_driver.py dual 128,197,768,3072 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 1 -c 1 \
  -o gpurun_out/tr/prof_acbp python tools/prof_driver.py acbp 128,197,3072,768 2 > /dev/null 2>&1
timeout 300 ncu --set full --clock-control none -k regex:"gemm_i8|tma_tile" -s 0 -c 4 \
  -o gpurun_out/tr/prof_conv python tools/conv_profile.py > /dev/null 2>&1
python tools/prof_summarize.py --round ${ROUND:-r01}_tr --out gpurun_out/tr_summary --reps gpurun_out/tr \
  --launches none > gpurun_out/tr_summary.log 2>&1
ncu -i gpurun_out/tr/prof_dual.ncu-rep --page source --csv --print-source sass > gpurun_out/tr_summary/dual_sass.csv 2>/dev/null
gzip -f gpurun_out/tr_summary/dual_sass.csv
rm -rf gpurun_out/tr
du -sh gpurun_out; ls -la gpurun_out/tr_summary
