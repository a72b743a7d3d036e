#!/bin/bash
# config 0 (w1 kernel) variants
run() {
  python bench.py --config 0 --steps 5 --warmup 3 --no-cpu --e2e-steps 2 > /tmp/o0.json 2>/tmp/o0.err
  python -c "import json; d=json.load(open('/tmp/o0.json')); r=d['roofline']; print('$1', round(d['value'],1), round(d['e2e']['value'],1), round(r['avg_launch_ms']*1000,2), 'us')" || tail -3 /tmp/o0.err
}
for i in 1 2; do
run default
for f in paper_2211_00805_b200/lib/variants/*.so; do GS_LIB=$f run $f; done
done
