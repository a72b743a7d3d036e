#!/bin/bash
# config 2 (narrow rows, R^30 kNN graph): CM + degree windows vs a recursive-bisection order
run() {
  python bench.py --config 2 --steps 2 --warmup 1 --sweeps 10 --no-cpu --e2e-steps 1 > /tmp/o2.json 2>/tmp/o2.err
  python -c "import json; d=json.load(open('/tmp/o2.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o2.err
}
run cm
GS_BENCH_ORDER=bisect run bisect64
