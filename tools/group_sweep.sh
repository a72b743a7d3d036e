#!/bin/bash
# config 1: 64-column groups vs two 32-column groups, launched together or group after group
run() {
  python bench.py --steps 2 --warmup 1 --sweeps 20 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],2), round(r['avg_launch_ms']*1000,1), 'us/launch', round(r['frac'],3), 'fp32', round((d.get('fp32_mode') or {}).get('value') or 0, 1))" || tail -3 /tmp/o.err
}
run gw64
GS_MAX_GW=32 run gw32
GS_MAX_GW=32 GS_SEQ_GROUPS=1 run gw32_seq
GS_MAX_GW=16 GS_SEQ_GROUPS=1 run gw16_seq
run gw64
