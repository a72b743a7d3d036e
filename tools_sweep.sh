#!/bin/bash
# tuning sweep: time the step kernel of each library variant (short bench runs; extra bench args in $ARGS)
run() {
  python bench.py --steps 2 --warmup 1 --sweeps ${SWEEPS:-20} --no-cpu --e2e-steps 1 --timing-period 1 $ARGS > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', '${GS_RPC}', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3), (d.get('fp32_mode') or {}).get('value'))" || tail -3 /tmp/o.err
}
run default
for f in paper_2211_00805_b200/lib/variants/*.so; do [ -e "$f" ] && GS_LIB=$f run $f; done
run default
for f in paper_2211_00805_b200/lib/variants/*.so; do [ -e "$f" ] && GS_LIB=$f run $f; done
