#!/bin/bash
# usage: gpurun -- bash tools/coop_ab.sh TAG : COOP on/off A/B on the small-batch configs
TAG=${1:-c}
mkdir -p gpurun_out
for co in 1 0; do
  export DIFFMPM_COOP=$co
  timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg2_co$co.json 2> gpurun_out/${TAG}_cfg2_co$co.err
  for E in 128 256; do
    timeout 300 python bench.py --envs $E --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg4_e${E}_co$co.json 2> gpurun_out/${TAG}_cfg4_e${E}_co$co.err
  done
done
