#!/bin/bash
# usage: gpurun -- bash tools/pdl_ab.sh TAG : GPU tests, then PDL on/off A/B (alternating, twice) per config
TAG=${1:-pdl}
mkdir -p gpurun_out
bash tools/gpu_tests.sh $TAG
for cfg in "--config 1 --steps 10" "--config 2 --steps 3" "--envs 128 --steps 3" "--steps 3"; do
  n=$(echo $cfg | tr -d ' -')
  for rep in a b; do
    for pdl in 1 0; do
      export DIFFMPM_PDL=$pdl
      timeout 600 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}_pdl${pdl}$rep.json 2> gpurun_out/${TAG}_${n}_pdl${pdl}$rep.err
    done
  done
done
unset DIFFMPM_PDL
