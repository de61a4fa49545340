#!/bin/bash
# Round profile captures on one B200 (run under gpurun from the repo root).
# Outputs land in gpurun_out/; tools/prof_summarize.py turns them into profiles/.
set -u
mkdir -p gpurun_out
# 1. every launch of one ViT-B/16 HLQ training step (cold-cache, serialised: shares, not absolutes)
HLQ_BENCH_MIN_WARMUP_S=0 timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none \
  --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-extras > gpurun_out/launches_bench.log 2>&1
# 2. the dominant kernel class: the fused transform (fc1 gy, dual, one cooperative launch)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 1 -c 1 \
  -o gpurun_out/prof_dual python tools/prof_driver.py dualcs 128,197,768,3072 2 > /dev/null 2>&1
# (acbp: launches 0-2 are the driver's setup transforms; -s 3 = the first ACBP of the loop)
timeout 300 ncu --set full --clock-control none --import-source on -k regex:tma_tile_kernel -s 3 -c 1 \
  -o gpurun_out/prof_acbp python tools/prof_driver.py acbp 128,197,3072,768 2 > /dev/null 2>&1
# 3. GEMMs as the training path plans them (fc1 dX, fc1 dW, fc2 dX)
for g in gemm_dx gemm_dw; do
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 1 -c 1 \
    -o gpurun_out/prof_fc1_$g python tools/prof_driver.py $g 128,197,768,3072 2 > /dev/null 2>&1
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_i8 -s 1 -c 1 \
  -o gpurun_out/prof_fc2_gemm_dx python tools/prof_driver.py gemm_dx 128,197,3072,768 2 > /dev/null 2>&1
# the fused dW + dX CTA-pair launch the training path issues for fc2 (and fc1)
for s in 128,197,3072,768 128,197,768,3072; do
  tag=$( [ $s = 128,197,3072,768 ] && echo fc2 || echo fc1 )
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:gemm_i8_2sm -s 1 -c 1 \
    -o gpurun_out/prof_${tag}_gemm_pair python tools/prof_driver.py gemm_pair $s 2 > /dev/null 2>&1
done
# 4. conv (BASELINE config b): implicit-GEMM dgrad and the im2col ACBP
timeout 300 ncu --set full --clock-control none -k regex:"gemm_i8|tma_tile" -s 0 -c 4 \
  -o gpurun_out/prof_conv python tools/conv_profile.py > /dev/null 2>&1
# 5. batched weight codes (49 ViT-B/16 weights)
timeout 300 ncu --set full --clock-control none -k regex:weight_codes -s 1 -c 1 \
  -o gpurun_out/prof_wcodes python -c "
import torch,sys; sys.path.insert(0,'.')
from paper_2406_15102_b200 import ops
ws=[torch.randn(o,i,device='cuda') for o,i in [(2304,768),(768,768),(3072,768),(768,3072)]*12+[(1000,768)]]
for _ in range(2): ops.quant_weights(ws,4)
torch.cuda.synchronize()" > /dev/null 2>&1
# summarise on the box (ncu is here) and keep gpurun_out/ under the 64 MiB copy-back limit
python tools/prof_summarize.py --round ${ROUND:-r01} --out gpurun_out/prof_summary > gpurun_out/prof_summary.log 2>&1
mkdir -p gpurun_out/reps
for f in gpurun_out/prof_*.ncu-rep; do
  if [ $(stat -c %s "$f") -lt 12000000 ]; then mv "$f" gpurun_out/reps/; else rm -f "$f"; fi
done
gzip -f gpurun_out/launches.csv
du -sh gpurun_out; ls -la gpurun_out/ gpurun_out/prof_summary gpurun_out/reps
