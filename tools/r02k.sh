for c in 2 4s; do echo "config $c"; GS_WIN_VERBOSE=1 timeout 300 python tools/prof_apply.py $c 1 2>&1 | grep -E 'gs_win|apply done'; done
timeout 300 ncu --set full --clock-control none -k regex:k_cheb_win -s 3 -c 2 -o gpurun_out/r02k_win_c2 python tools/prof_apply.py 2 1 > gpurun_out/r02k_ncu.log 2>&1; echo ncu=$?
