#!/bin/bash
# usage: gpurun -- bash tools/r2_prof2.sh TAG CONFIG ENVS CTRL K1 [K2 ...]
# ncu --set full of the named kernels (steady state: 6th launch) -> details/raw CSV
# + SASS source-page CSV (gz; tools/sass_lines.py maps it to CUDA lines).  No .ncu-rep kept (64 MiB cap).
mkdir -p gpurun_out
TAG=$1; CFG=$2; ENVS=$3; CTRL=$4; shift 4
for K in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}(<|$)" -s 6 -c 1 -o /tmp/${TAG}_${K} -f python tools/prof_rollout.py --config $CFG --envs $ENVS --ctrl $CTRL > gpurun_out/${TAG}_${K}.log 2>&1
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > gpurun_out/${TAG}_${K}_sass.csv.gz
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/prof_rollout.py --config $CFG --envs $ENVS --ctrl $CTRL > gpurun_out/${TAG}_launches.csv 2>&1
du -sh gpurun_out
