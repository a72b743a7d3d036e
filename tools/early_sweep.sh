#!/bin/bash
# own-row operands loaded before the gathers (GS_EARLY_OWN) on the unstaged layouts: config 2 / 3
run() {
  python bench.py $ARGS --steps 2 --warmup 1 --no-cpu --e2e-steps 1 > /tmp/o.json 2>/tmp/o.err
  python -c "import json,sys; d=json.load(open('/tmp/o.json')); r=d['roofline']; print('$1', round(d['value'],3), round(r['avg_launch_ms']*1000,1), 'us', round(r['frac'],3))" || tail -3 /tmp/o.err
}
for c in 2 3; do
  export ARGS="--config $c --sweeps 10"
  run "c$c early"
  for f in paper_2211_00805_b200/lib/variants/*.so; do GS_LIB=$f run "c$c $f"; done
done
