#!/bin/bash
# usage: gpurun -- bash tools/so_ab.sh TAG variant.so : default build vs a library variant, alternating, on 128 envs, cfg2, cfg4 (4 control steps) and cfg1
TAG=$1; V=$2
mkdir -p gpurun_out
for cfg in "--envs 128 --steps 3" "--config 2 --steps 3" "--ctrl 4 --steps 3" "--config 1 --steps 10"; do
  n=$(echo $cfg | tr -d ' -')
  for rep in a b; do
    timeout 600 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}_def$rep.json 2>/dev/null
    DIFFMPM_SO=$V timeout 600 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}_var$rep.json 2>/dev/null
  done
done
