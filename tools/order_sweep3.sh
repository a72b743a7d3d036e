#!/bin/bash
# config 3 (n = 2e7, fp32, B = 1): CM order vs a 3-D Morton order of the points
for o in "" morton; do
  GS_BENCH_ORDER=$o python bench.py --config 3 --steps 2 --warmup 1 --sweeps 20 --no-cpu --e2e-steps 1 > /tmp/o3.json 2>/tmp/o3.err
  python -c "import json; d=json.load(open('/tmp/o3.json')); r=d['roofline']; print('order=${o:-cm}', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o3.err
done
