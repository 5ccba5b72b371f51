#!/bin/bash
# Round-2 evidence: regime comparison on the runtime, VGG 7-1 sharded vs one-shot replica reduction,
# ncu --set full of the three MLP GEMMs and the two attention kernels.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
what=${1:-all}
if [[ $what == compare || $what == all ]]; then
  timeout 900 python -m paper_1806_03377_b200 compare profiles/layer_profiles/mlp8192_profile.json \
    --model mlp:8192:16:2048:bf16 --machines 8 --minibatches 32 --lr 1e-5 --out-dir gpurun_out/compare_mlp \
    > gpurun_out/compare_mlp.log 2>&1; echo "compare mlp rc=$?"; tail -8 gpurun_out/compare_mlp.log
  timeout 900 python -m paper_1806_03377_b200 compare profiles/layer_profiles/vgg16_profile.json \
    --model vgg16:32 --machines 8 --minibatches 56 --lr 1e-4 --bandwidth 12.5e9 --out-dir gpurun_out/compare_vgg \
    > gpurun_out/compare_vgg.log 2>&1; echo "compare vgg rc=$?"; tail -8 gpurun_out/compare_vgg.log
fi
if [[ $what == reduce || $what == all ]]; then
  for sh in 1 0; do
    PD_SHARDED_REDUCE=$sh timeout 600 python bench.py --workload vgg --no-cpu-baseline --steps 3 --warmup 2 \
      > gpurun_out/vgg_sharded_$sh.json 2>/dev/null
    python -c "import json;d=json.loads(open('gpurun_out/vgg_sharded_$sh.json').read().strip().splitlines()[-1]);print('sharded=$sh', round(d['value'],1), d['unit'], d['kernel_time_ms_serial_step'].get('update'), d['clocks']['sm_mhz'])"
  done
fi
if [[ $what == ncu || $what == all ]]; then
  for spec in "fwd 3" "dgrad 16" "wgrad 29"; do
    set -- $spec
    timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s $2 -c 1 \
      -o gpurun_out/r02b_prof_$1 -f python tools/gemm_bench.py > gpurun_out/ncu_$1.log 2>&1; tail -1 gpurun_out/ncu_$1.log
    ncu -i gpurun_out/r02b_prof_$1.ncu-rep --page details --csv > gpurun_out/r02b_prof_$1.details.csv 2>/dev/null
    ncu -i gpurun_out/r02b_prof_$1.ncu-rep --page raw --csv > gpurun_out/r02b_prof_$1.raw.csv 2>/dev/null
    gzip -f gpurun_out/r02b_prof_$1.raw.csv; rm -f gpurun_out/r02b_prof_$1.ncu-rep
  done
  bash tools/gpu_r02_attn_prof.sh
fi
