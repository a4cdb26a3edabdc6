#!/bin/bash
# usage: gpurun -- bash tools/r2_final2.sh TAG : every bench line (tools/r2_full.sh) + the cfg1 launch list (PDL chain)
TAG=${1:-g}
bash tools/r2_full.sh $TAG
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_cfg1_launches.csv python bench.py --config 1 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_cfg1_ncu.log 2>&1
