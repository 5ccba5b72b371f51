#!/bin/bash
# cfg5 evidence on one B200: MLP-8192 stage sweep (2/4/8 straight stages, all on one GPU) and the
# same-device IPC hand-off microbench (two ranks sharing the GPU).  Outputs under gpurun_out/cfg5/.
set -u
mkdir -p gpurun_out/cfg5
for s in 2 4 8; do
  PD_BENCH_WATCHDOG_S=300 timeout 600 python bench.py --workload mlp --stages $s --no-cpu-baseline \
    --steps 5 --warmup 3 > gpurun_out/cfg5/stages_$s.json 2> gpurun_out/cfg5/stages_$s.err
  tail -1 gpurun_out/cfg5/stages_$s.json | cut -c1-200
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
  --master-port 29555 tools/p2p_bench.py > gpurun_out/cfg5/p2p.json 2> gpurun_out/cfg5/p2p.err
tail -c 600 gpurun_out/cfg5/p2p.json
