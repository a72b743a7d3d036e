#!/bin/bash
# tuning: degree-sorted window size sigma on configs 1 and 2 (step kernel average)
for sg in 0 64 256; do
  GS_SIGMA=$sg python bench.py --steps 1 --warmup 1 --sweeps 20 --no-cpu --no-fp32 --e2e-steps 1 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg1 sigma=$sg', round(d['roofline']['avg_launch_ms']*1000,1), 'us')"
  GS_SIGMA=$sg python bench.py --config 2 --n 200000 --steps 1 --warmup 1 --sweeps 20 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg2(n=200k) sigma=$sg', round(d['roofline']['avg_launch_ms']*1000,1), 'us', round(d['roofline']['frac'],3))"
done
