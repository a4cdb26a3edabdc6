#!/bin/bash
# usage: gpurun -- bash tools/r2_bench.sh TAG  : default bench (cfg4) + cfg3 (2 ctrl) + cfg1 + cfg2
TAG=${1:-b}
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/${TAG}_cfg4.json 2> gpurun_out/${TAG}_cfg4.err
timeout 600 python bench.py --config 3 --ctrl 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg3.json 2> gpurun_out/${TAG}_cfg3.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg1.json 2> gpurun_out/${TAG}_cfg1.err
timeout 300 python bench.py --config 2 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
