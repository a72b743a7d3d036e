#!/bin/bash
# One measurement pass on a B200 (run under gpurun from the repo root): GPU tests, smoke, bench
# lines for configs 0-3, the config-1 launch list and ncu --set full captures of the step kernel
# (config 1 wide layout, config 2 narrow layout). Output: gpurun_out/m_*.
set -u
O=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/m_gpu_tests.log 2>&1; echo "exit $?" >> $O/m_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > $O/m_smoke.log 2>&1; echo "exit $?" >> $O/m_smoke.log
for c in 1 0 2 3; do
  timeout 900 python bench.py --config $c > $O/m_bench_c$c.json 2> $O/m_bench_c$c.err
done
SHORT="python bench.py --steps 1 --warmup 0 --sweeps 1 --no-cpu --e2e-steps 1 --no-fp32"
SHORT2="python bench.py --config 2 --steps 1 --warmup 0 --sweeps 1 --no-cpu --e2e-steps 1"
$SHORT > $O/m_plain1.log 2>&1 && $SHORT2 > $O/m_plain2.log 2>&1 && {
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/m_launches.csv $SHORT > $O/m_ncu_launch.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_cheb_step -s 10 -c 3 -o $O/m_c1_step $SHORT > $O/m_ncu_c1.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:k_cheb_step -s 5 -c 3 -o $O/m_c2_step $SHORT2 > $O/m_ncu_c2.log 2>&1
}
echo done > $O/m_done
