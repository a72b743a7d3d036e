#!/bin/bash
# Round-2 measurement pass (one B200): bench lines, ncu captures of the dominant kernels, launch list.
set -x
T=${TAG:-r02z}
timeout 900 python bench.py > gpurun_out/${T}_bench_c1.json 2> gpurun_out/${T}_bench_c1.err; echo bench_c1=$?
timeout 300 python bench.py --config 0 > gpurun_out/${T}_bench_c0.json 2> gpurun_out/${T}_bench_c0.err; echo bench_c0=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_cheb_win -s 3 -c 3 -o gpurun_out/${T}_win_c1 python tools/prof_apply.py 1 > gpurun_out/${T}_ncu_win.log 2>&1; echo ncu_win=$?
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_sk_persist -c 1 -o gpurun_out/${T}_persist_c0 python tools/prof_c0.py 1 > gpurun_out/${T}_ncu_persist.log 2>&1; echo ncu_persist=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${T}_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu --no-fp32 --no-legs > gpurun_out/${T}_ncu_launches.log 2>&1; echo ncu_launches=$?
