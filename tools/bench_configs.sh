#!/bin/bash
# bench lines for configs 2, 3, 4 (one B200)
T=${TAG:-r02}
timeout 900 python bench.py --config 2 > gpurun_out/${T}_bench_c2.json 2> gpurun_out/${T}_bench_c2.err; echo c2=$?
timeout 900 python bench.py --config 3 > gpurun_out/${T}_bench_c3.json 2> gpurun_out/${T}_bench_c3.err; echo c3=$?
timeout 1500 python bench.py --config 4 --steps 1 --warmup 1 > gpurun_out/${T}_bench_c4.json 2> gpurun_out/${T}_bench_c4.err; echo c4=$?
