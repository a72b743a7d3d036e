#!/bin/bash
# Variant sweep of the windowed step kernel on config 1 (bench.py, no CPU / fp32 legs).
# Usage: bash tools/win_sweep.sh tag variant1 variant2 ...   (variants/lib_<v>.so; "base" = default build,
# "off" = GS_WIN=0, "A=1,B=2" = the default build under those environment variables)
tag=$1; shift
for v in "$@"; do
  if [ "$v" = base ]; then env=""; elif [ "$v" = off ]; then env="GS_WIN=0"; elif [[ "$v" == *=* ]]; then env="${v//,/ }"; else env="GS_LIB=variants/lib_$v.so"; fi
  env $env timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu --no-fp32 > gpurun_out/${tag}_$v.json 2> gpurun_out/${tag}_$v.err
  python - "$v" gpurun_out/${tag}_$v.json <<'PY'
import json, sys
try:
    d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
    r = d["roofline"]
    print(f"{sys.argv[1]:8s} value={d['value']:.2f} step_us={r['avg_launch_ms']*1e3:.1f} frac={r['frac']:.3f} lb_frac={r['lower_bound_from_timed_region']['frac']:.3f} sm_mhz={d['clocks']['sm_mhz']}")
except Exception as e:
    print(sys.argv[1], "failed", e)
PY
done
