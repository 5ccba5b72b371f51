#!/bin/bash
# Round-2 evidence run (one GPU): compute-sanitizer over the pipeline protocol, ncu launch list of
# the bench command, ncu --set full of the three bench GEMMs.  Outputs under gpurun_out/.
set -u
mkdir -p gpurun_out
what=${1:-all}
if [[ $what == sanitize || $what == all ]]; then
  for tool in memcheck racecheck synccheck; do
    timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_target.py mlp rep conv gpt \
      > gpurun_out/sanitize_$tool.log 2>&1
    echo "== $tool rc=$?"; grep -E "ERROR SUMMARY|sanitize target|Error|error" gpurun_out/sanitize_$tool.log | head -8
    head -c 300000 gpurun_out/sanitize_$tool.log > gpurun_out/sanitize_$tool.head.log; rm -f gpurun_out/sanitize_$tool.log
  done
fi
if [[ $what == ncu || $what == all ]]; then
  timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv \
    --log-file gpurun_out/launches_r02.csv python bench.py --steps 1 --warmup 1 --minibatches 32 --no-cpu-baseline \
    --e2e-steps 1 > gpurun_out/ncu_bench.log 2>&1; tail -2 gpurun_out/ncu_bench.log
  for spec in "fwd 3" "dgrad 16" "wgrad 29"; do
    set -- $spec
    timeout -s KILL 300 ncu --set full --clock-control none --import-source on -k regex:k_gemm_tc -s $2 -c 1 \
      -o gpurun_out/r02_prof_$1 -f python tools/gemm_bench.py > gpurun_out/ncu_$1.log 2>&1; tail -1 gpurun_out/ncu_$1.log
    ncu -i gpurun_out/r02_prof_$1.ncu-rep --page raw --csv > gpurun_out/r02_prof_$1.raw.csv 2>/dev/null
    ncu -i gpurun_out/r02_prof_$1.ncu-rep --page details --csv > gpurun_out/r02_prof_$1.details.csv 2>/dev/null
    ncu -i gpurun_out/r02_prof_$1.ncu-rep --page source --csv --print-source sass > gpurun_out/r02_prof_$1.sass.csv 2>/dev/null
    gzip -f gpurun_out/r02_prof_$1.sass.csv; ls -la gpurun_out/r02_prof_$1*; rm -f gpurun_out/r02_prof_$1.ncu-rep
  done
  du -sh gpurun_out
fi
