#!/bin/bash
# usage: gpurun -- bash tools/cg_pdl_ab.sh TAG : COOP group size 2 vs 4 with launch chaining (cfg2, 128 envs), alternating
TAG=${1:-cg}
mkdir -p gpurun_out
for cfg in "--config 2 --steps 3" "--envs 128 --steps 3"; do
  n=$(echo $cfg | tr -d ' -')
  for rep in a b; do
    for cg in 2 4; do
      DIFFMPM_COOP_CG=$cg timeout 600 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}_cg$cg$rep.json 2>/dev/null
    done
  done
done
