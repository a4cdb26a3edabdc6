#!/bin/bash
# usage: gpurun -- bash tools/r2_quick.sh TAG : GPU tests + smoke + short benches (cfg4, cfg4 x128, cfg2, cfg1)
TAG=${1:-q}
bash tools/gpu_tests.sh $TAG
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg4.json 2> gpurun_out/${TAG}_cfg4.err
timeout 300 python bench.py --envs 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg4_e128.json 2>gpurun_out/${TAG}_cfg4_e128.err
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg2.json 2>gpurun_out/${TAG}_cfg2.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg1.json 2>gpurun_out/${TAG}_cfg1.err
