#!/bin/bash
# One GPU session: tests, smoke, bench, ncu launch list + full capture of the top GEMM.
# Usage (under gpurun): bash tools/gpu_round.sh [tests|bench|ncu|all]
set -u
mkdir -p gpurun_out
what=${1:-all}
if [[ $what == tests || $what == all ]]; then
  timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | grep -v Warning | tail -30 > gpurun_out/gpu_tests.log
  timeout -s KILL 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
  tail -3 gpurun_out/gpu_tests.log; cat gpurun_out/smoke.log
fi
if [[ $what == bench || $what == all ]]; then
  timeout -s KILL 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -5 gpurun_out/bench.err; cat gpurun_out/bench.json
  timeout -s KILL 600 python bench.py --serial off --no-cpu-baseline > gpurun_out/bench_multistream.json 2>&1; cat gpurun_out/bench_multistream.json
  timeout -s KILL 200 python tools/gemm_bench.py 2048 8192 > gpurun_out/gemm_bench.log 2>&1; cat gpurun_out/gemm_bench.log
  timeout -s KILL 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; cat gpurun_out/bench_ref.json
fi
if [[ $what == ncu || $what == all ]]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 \
    > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 3 -c 1 \
    -o gpurun_out/prof_fwd -f python tools/gemm_bench.py > gpurun_out/ncu_fwd.log 2>&1; tail -2 gpurun_out/ncu_fwd.log
  timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s 29 -c 1 \
    -o gpurun_out/prof_wgrad -f python tools/gemm_bench.py > gpurun_out/ncu_wgrad.log 2>&1; tail -2 gpurun_out/ncu_wgrad.log
fi
