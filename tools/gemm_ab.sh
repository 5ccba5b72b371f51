#!/bin/bash
# A/B of the 1-CTA and CTA-pair GEMM: correctness tests + timing, each under its own timeout.
mkdir -p gpurun_out
for cg in 2 1 0; do
  echo "== PD_GEMM_CG=$cg"
  PD_GEMM_CG=$cg timeout -s KILL 240 python -m pytest tests/test_gemm_gpu.py tests/test_layer_step_gpu.py -q -x 2>&1 | tail -2
  PD_GEMM_CG=$cg timeout -s KILL 120 python tools/gemm_bench.py 2048 8192
done
