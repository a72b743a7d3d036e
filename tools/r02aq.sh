for v in base bulk; do
  if [ $v = base ]; then e=""; else e="GS_LIB=variants/lib_$v.so"; fi
  echo "config 2 narrow on window, $v"; env $e GS_WIN_MIN_BYTES=32 timeout 300 python tools/prof_apply.py 2 3 2>&1 | tail -1
done
bash tools/win_sweep.sh r02aq base bulk
