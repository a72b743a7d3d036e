#!/bin/bash
# per-call workspace cost: default mempool release (GS_POOL_KEEP=0) vs keeping pool memory
for keep in 0 1; do
  for c in 1 3; do
    GS_POOL_KEEP=$keep python bench.py --config $c --steps 3 --warmup 3 --no-cpu --no-fp32 > /tmp/p.json 2>/tmp/p.err
    python -c "import json; d=json.load(open('/tmp/p.json')); print('keep=$keep config $c value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3))" || tail -3 /tmp/p.err
  done
done
