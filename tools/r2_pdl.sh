#!/bin/bash
# usage: gpurun -- bash tools/r2_pdl.sh TAG : GPU tests + smoke, default benches, PDL A/B at 128 envs
TAG=${1:-q}
bash tools/gpu_tests.sh $TAG
for cfg in "--config 1 --steps 10" "--config 2 --steps 3" "--envs 128 --steps 3" "--steps 3" "--config 3 --steps 2"; do
  n=$(echo $cfg | tr -d ' -')
  timeout 600 python bench.py $cfg --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${n}.json 2> gpurun_out/${TAG}_${n}.err
done
for pdl in 0 1; do
  DIFFMPM_PDL=$pdl timeout 600 python bench.py --envs 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_e128_pdl$pdl.json 2> gpurun_out/${TAG}_e128_pdl$pdl.err
done
