#!/bin/bash
# usage: gpurun -- bash tools/r2_full.sh TAG : every bench line of the round (outputs -> gpurun_out/TAG_*.json)
#   default bench (cfg4, e2e + cpu baseline), the reference arm, cfg3 full horizon,
#   cfg2, cfg1, cfg5 (SAPO iteration), cfg4 at 128 envs (a strong-scaling shard)
TAG=${1:-full}
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/${TAG}_cfg4.json 2> gpurun_out/${TAG}_cfg4.err
timeout 900 python bench.py --impl reference > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg3.json 2> gpurun_out/${TAG}_cfg3.err
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg2.json 2> gpurun_out/${TAG}_cfg2.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg1.json 2> gpurun_out/${TAG}_cfg1.err
timeout 900 python bench.py --config 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg5.json 2> gpurun_out/${TAG}_cfg5.err
timeout 300 python bench.py --envs 128 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_cfg4_e128.json 2> gpurun_out/${TAG}_cfg4_e128.err
