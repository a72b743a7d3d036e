for lib in "" "GS_LIB=variants/lib_s1m4.so"; do
for pf in "0 0" "4 0" "4096 4096" "16384 16384" "65536 65536" "0 16384"; do
set -- $pf
echo -n "$lib pf $1 $2: "
env $lib GS_LANE_PF_BACK=$1 GS_LANE_PF_FWD=$2 timeout 900 python tools/prof_apply.py 3 3 2>&1 | tail -n 1
done; done
