#!/bin/bash
# tuning sweep: time the step kernel of each library variant on config 1 (short runs)
run() {
  python bench.py --steps 2 --warmup 1 --sweeps 20 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o.err
}

run default
for f in paper_2211_00805_b200/lib/variants/*.so; do GS_LIB=$f run $f; done
