timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_properties.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/t_blk.log 2>&1
bash tools_sweep.sh > gpurun_out/sweep_blk.txt 2>&1
GS_BLK=0 bash tools_sweep.sh 2>&1 | head -1 | sed 's/^/GS_BLK=0 /' >> gpurun_out/sweep_blk.txt
