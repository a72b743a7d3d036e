#!/bin/bash
# config 3 step-kernel variants: env toggles and GS_LIB builds, short runs
run() {
  python bench.py --config 3 --steps 2 --warmup 1 --sweeps 10 --no-cpu --e2e-steps 1 > /tmp/o3.json 2>/tmp/o3.err
  python -c "import json; d=json.load(open('/tmp/o3.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o3.err
}
for i in 1 2; do
run default
GS_RPC=1 run rpc1
for f in paper_2211_00805_b200/lib/variants/*.so; do [ -e "$f" ] && GS_LIB=$f run $f; done
done
