#!/bin/bash
# A/B of the staged one-row-per-lane kernel (k_cheb_lane) on config-3 shapes:
# tools/lane_ab.sh "cfgs" variant...   variant: base | off (GS_LANE=0) | <name> (variants/lib_<name>.so)
cfgs=$1; shift
for cfg in $cfgs; do
  for v in "$@"; do
    if [ "$v" = base ]; then env=""; elif [ "$v" = off ]; then env="GS_LANE=0"; elif [[ "$v" == *=* ]]; then env="${v//,/ }"; else env="GS_LIB=variants/lib_$v.so"; fi
    echo -n "config $cfg $v: "
    env $env timeout 900 python tools/prof_apply.py $cfg 3 2>&1 | tail -1
  done
done
