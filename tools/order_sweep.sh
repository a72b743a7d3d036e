#!/bin/bash
# locality-order experiment: config 1 step time under host-computed orders (gs_filter_set_order)
run() {
  python bench.py --steps 2 --warmup 1 --sweeps 20 --no-cpu --e2e-steps 1 --timing-period 1 $ARGS > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3), (d.get('fp32_mode') or {}).get('value'))" || tail -3 /tmp/o.err
}
run cm
GS_BENCH_ORDER=morton run morton
GS_BENCH_ORDER=bisect run bisect64
GS_BENCH_ORDER=bisect GS_BENCH_LEAF=32 run bisect32
GS_BENCH_ORDER=bisect GS_BENCH_LEAF=256 run bisect256
run cm
