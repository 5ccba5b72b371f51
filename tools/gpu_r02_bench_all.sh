mkdir -p gpurun_out/e2e
for w in vgg gpt mlp; do
  PD_BENCH_WATCHDOG_S=600 timeout 900 python bench.py --workload $w > gpurun_out/e2e/bench_$w.json 2> gpurun_out/e2e/bench_$w.err
  python -c "
import json;d=json.loads(open('gpurun_out/e2e/bench_$w.json').read().strip().splitlines()[-1])
print('$w', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
