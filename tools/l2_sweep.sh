#!/bin/bash
# L2 persistence experiment (GS_L2_PERSIST) on configs 1 and 2
run() {
  python bench.py --steps 2 --warmup 1 --sweeps ${SWEEPS:-20} --no-cpu --e2e-steps 1 --timing-period 1 $ARGS > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3), (d.get('fp32_mode') or {}).get('value'))" || tail -3 /tmp/o.err
}
for p in 0 1 0 1; do GS_L2_PERSIST=$p run "c1 persist=$p"; done
for p in 0 1; do SWEEPS=10 ARGS="--config 2" GS_L2_PERSIST=$p run "c2 persist=$p"; done
