#!/bin/bash
# A/B of the sliced step kernel on apply shapes: tools/sell_ab.sh "cfgs" variant...
# variant: base | off (GS_SELL=0) | <name> (variants/lib_<name>.so) | A=1,B=2 (environment)
cfgs=$1; shift
for cfg in $cfgs; do
  for v in "$@"; do
    if [ "$v" = base ]; then env=""; elif [ "$v" = off ]; then env="GS_SELL=0"; elif [[ "$v" == *=* ]]; then env="${v//,/ }"; else env="GS_LIB=variants/lib_$v.so"; fi
    echo -n "config $cfg $v: "
    env $env timeout 600 python tools/prof_apply.py $cfg 3 2>&1 | tail -1
  done
done
