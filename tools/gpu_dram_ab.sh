#!/bin/bash
# DRAM bytes of the MLP-8192 forward / dgrad GEMMs with and without the evict-first B policy.
for bs in 0 1; do
  PD_B_STREAM=$bs ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
    -k regex:k_gemm_tc -s 10 -c 6 --csv python tools/gemm_bench.py 2>/dev/null \
    | python -c "
import csv,sys
rows=[r for r in csv.reader(sys.stdin) if len(r)>10]
h=rows[0]; k=h.index('Kernel Name'); m=h.index('Metric Name'); v=h.index('Metric Value'); u=h.index('Metric Unit')
for r in rows[1:]: print('b_stream=$bs', r[k][:40], r[m], r[v], r[u])
"
  PD_B_STREAM=$bs python tools/gemm_bench.py
done
