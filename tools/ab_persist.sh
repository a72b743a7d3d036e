#!/bin/bash
# A/B of the resident-grid plain steps (GS_PERSIST) on configs 1-4 (short runs)
j() { python -c "import json,sys; d=json.loads(open('/tmp/o.json').read().strip().split('\n')[-1]); print('$1', round(d['value'],3), round(d['roofline']['avg_launch_ms']*1000,1), 'us')" || tail -2 /tmp/o.err; }
for P in 0 1; do
  export GS_PERSIST=$P
  python bench.py --steps 2 --warmup 3 --sweeps 40 --no-cpu --no-fp32 --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err; j "c1 persist=$P"
  python bench.py --config 2 --steps 2 --warmup 3 --sweeps 20 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err; j "c2 persist=$P"
  python bench.py --config 3 --n 4000000 --steps 2 --warmup 3 --sweeps 20 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err; j "c3 persist=$P"
  python bench.py --config 4 --n 400000 --steps 2 --warmup 3 --sweeps 50 --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err; j "c4 persist=$P"
done
