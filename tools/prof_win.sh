set -x
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_cheb_win -s 3 -c 3 -o gpurun_out/${TAG:-r02g}_win_c1 python tools/prof_apply.py 1 > gpurun_out/${TAG:-r02g}_ncu.log 2>&1
echo ncu_rc=$?
tail -3 gpurun_out/${TAG:-r02g}_ncu.log
