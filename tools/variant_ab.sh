#!/bin/bash
# usage: gpurun -- bash tools/variant_ab.sh TAG lib1 [lib2 ...] : cfg4 (4 control steps) per library variant + the default build
TAG=$1; shift
mkdir -p gpurun_out
timeout 600 python bench.py --ctrl 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_default.json 2>/dev/null
for so in "$@"; do
  n=$(basename $so .so)
  DIFFMPM_SO=$so timeout 600 python bench.py --ctrl 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_$n.json 2>/dev/null
done
