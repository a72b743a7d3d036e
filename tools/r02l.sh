GS_LIB=variants/lib_cpa.so timeout 300 python -m pytest tests -m gpu -x -q -k "parity or config" > gpurun_out/r02l_tests.log 2>&1; echo tests_cpa=$?; tail -1 gpurun_out/r02l_tests.log
for v in base cpa; do
  if [ $v = base ]; then e=""; else e="GS_LIB=variants/lib_$v.so"; fi
  echo "config 2 $v"; env $e timeout 300 python tools/prof_apply.py 2 3 2>&1 | tail -1
done
bash tools/win_sweep.sh r02l base cpa
