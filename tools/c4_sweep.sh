#!/bin/bash
# config 4 layout (B = 16 fp64, 128-byte rows) variants on a 1e6-point instance
run() {
  python bench.py --config 4 --n 1000000 --steps 2 --warmup 1 --sweeps 10 --no-cpu --e2e-steps 1 > /tmp/o4.json 2>/tmp/o4.err
  python -c "import json; d=json.load(open('/tmp/o4.json')); r=d['roofline']; print('$1', round(d['value'],4), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o4.err
}
run default
for f in paper_2211_00805_b200/lib/variants/*.so; do [ -e "$f" ] && GS_LIB=$f run $f; done
