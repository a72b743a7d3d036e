#!/bin/bash
# A/B of the record kernel (k_cheb_rec) on the barycenter shapes:
# tools/rec_ab.sh "cfgs" variant...   variant: base | off (GS_REC=0) | <name> (variants/lib_<name>.so) | A=1,B=2
cfgs=$1; shift
for cfg in $cfgs; do
  for v in "$@"; do
    if [ "$v" = base ]; then env=""; elif [ "$v" = off ]; then env="GS_REC=0"; elif [[ "$v" == *=* ]]; then env="${v//,/ }"; else env="GS_LIB=variants/lib_$v.so"; fi
    echo -n "config $cfg $v: "
    env $env timeout 900 python tools/prof_apply.py $cfg 3 2>&1 | tail -n 1
  done
done
