timeout 400 python -m pytest tests -m gpu -x -q > gpurun_out/r02m_tests.log 2>&1; echo tests=$?; tail -1 gpurun_out/r02m_tests.log
for c in 2 4s; do echo "config $c"; GS_WIN_VERBOSE=1 timeout 300 python tools/prof_apply.py $c 3 2>&1 | grep -E 'gs_win\] row|apply done'; done
bash tools/win_sweep.sh r02m base
GS_WIN_MARGIN_DIV=8 bash tools/win_sweep.sh r02m8 base
GS_WIN_MARGIN_DIV=2 bash tools/win_sweep.sh r02m2 base
