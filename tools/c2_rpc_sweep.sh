#!/bin/bash
# row blocks per CTA for the narrow / 16-column layouts (GS_RPC) on config 2 and a 1e6-point config 4
run() {
  python bench.py $ARGS --steps 2 --warmup 1 --sweeps 10 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],4), round(r['avg_launch_ms']*1000,1), 'us')" || tail -3 /tmp/o.err
}
export ARGS="--config 2"
for i in 1 2; do run "c2 rpc1"; GS_RPC=4 run "c2 rpc4"; done
export ARGS="--config 4 --n 1000000"
run "c4 rpc1"; GS_RPC=4 run "c4 rpc4"
