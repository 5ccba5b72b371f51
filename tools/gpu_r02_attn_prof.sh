#!/bin/bash
# ncu --set full of the attention kernels (one launch each) + the SGD raster-band sweep.
set -u
mkdir -p gpurun_out

for k in k_attn_fwd_tc2 k_attn_bwd_tc; do
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 \
    -o gpurun_out/prof_$k -f python tools/attn_bench.py > gpurun_out/ncu_$k.log 2>&1; tail -1 gpurun_out/ncu_$k.log
  ncu -i gpurun_out/prof_$k.ncu-rep --page details --csv > gpurun_out/prof_$k.details.csv 2>/dev/null
  ncu -i gpurun_out/prof_$k.ncu-rep --page raw --csv > gpurun_out/prof_$k.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/prof_$k.sass.csv 2>/dev/null
  gzip -f gpurun_out/prof_$k.sass.csv gpurun_out/prof_$k.raw.csv
  rm -f gpurun_out/prof_$k.ncu-rep
done
ls -la gpurun_out
