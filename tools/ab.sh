#!/bin/bash
# A/B timing of library variants on the GPU box: bench.py (cfg4, 2 control
# steps; BENCH_ARGS overrides) once per .so.  usage: bash tools/ab.sh TAG so1 [so2 ...]
TAG=$1; shift
mkdir -p gpurun_out
for so in "$@"; do
  n=$(basename $so .so)
  DIFFMPM_SO=$so timeout 600 python bench.py ${BENCH_ARGS:---ctrl 2} --steps 2 --warmup 3 --no-e2e --no-cpu-baseline \
    > gpurun_out/${TAG}_${n}.json 2> gpurun_out/${TAG}_${n}.err
  echo "$n EXIT $?" >> gpurun_out/${TAG}_${n}.err
done
