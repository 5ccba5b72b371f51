#!/bin/bash
# End-of-round evidence on the final build (one GPU): ncu --set full of the three MLP-8192 bench
# GEMMs (tools/gemm_bench.py launches 3 / 16 / 29 = forward / dgrad / wgrad+SGD), the ncu launch
# list of the bench command, and ncu_traffic.json for bench.py's roofline.traffic.
set -u
mkdir -p gpurun_out
for spec in "fwd 3" "dgrad 16" "wgrad 29"; do
  set -- $spec
  timeout -s KILL 300 ncu --set full --clock-control none -k regex:k_gemm_tc -s $2 -c 1 \
    -o gpurun_out/fin_$1 -f python tools/gemm_bench.py > /dev/null 2>&1
  ncu -i gpurun_out/fin_$1.ncu-rep --page details --csv > gpurun_out/fin_$1.details.csv 2>/dev/null
  ncu -i gpurun_out/fin_$1.ncu-rep --page raw --csv > gpurun_out/fin_$1.raw.csv 2>/dev/null
  gzip -f gpurun_out/fin_$1.raw.csv; rm -f gpurun_out/fin_$1.ncu-rep
done
timeout -s KILL 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
  --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 1 --minibatches 32 --no-cpu-baseline \
  --e2e-steps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/fin_launches.csv 12 > gpurun_out/fin_launches_summary.txt
gzip -f gpurun_out/fin_launches.csv
cat gpurun_out/fin_launches_summary.txt
