#!/bin/bash
# ncu --set full of the small (768-wide) transforms: forward ACBP proj and the
# fc2-shape dual; source-level SASS CSVs summarised on the box.
set -u
mkdir -p gpurun_out/small
for what in acbp dual; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 3 -c 1 \
    -o gpurun_out/small/prof_$what python tools/prof_driver.py $what 128,197,768,768 3 > /dev/null 2>&1
  ncu -i gpurun_out/small/prof_$what.ncu-rep --page source --csv --print-source sass \
    > gpurun_out/small/${what}_sass.csv 2>/dev/null
  ncu -i gpurun_out/small/prof_$what.ncu-rep --page raw --csv > gpurun_out/small/${what}_raw.csv 2>/dev/null
  gzip -f gpurun_out/small/${what}_sass.csv gpurun_out/small/${what}_raw.csv
  rm -f gpurun_out/small/prof_$what.ncu-rep
done
ls -la gpurun_out/small
