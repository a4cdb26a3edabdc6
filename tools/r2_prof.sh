#!/bin/bash
# ncu --set full of the hot kernels (cfg4, 1024 envs, steady state) -> CSV summaries
# (+ one .ncu-rep), compute-sanitizer logs.  Output stays under 64 MiB.
mkdir -p gpurun_out
TAG=${1:-p}
KEEP=${2:-k_p2g}
for K in k_p2g k_g2p k_g2p_adj k_p2g_adj k_bin k_grid k_grid_adj k_cellsort; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^${K}(<|$)" -s 6 -c 1 -o /tmp/${TAG}_${K} -f python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 2 > gpurun_out/${TAG}_${K}.log 2>&1
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page details --csv > gpurun_out/${TAG}_${K}_details.csv 2>/dev/null
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page raw --csv > gpurun_out/${TAG}_${K}_raw.csv 2>/dev/null
  ncu -i /tmp/${TAG}_${K}.ncu-rep --page source --csv --print-source sass > /tmp/${TAG}_${K}_sass.csv 2>/dev/null
  gzip -c /tmp/${TAG}_${K}_sass.csv > gpurun_out/${TAG}_${K}_sass.csv.gz
  if [ "$K" == "$KEEP" ]; then cp /tmp/${TAG}_${K}.ncu-rep gpurun_out/; fi
done
if [ "$3" != "nosan" ]; then
timeout 900 compute-sanitizer --tool racecheck --racecheck-report analysis python tools/prof_rollout.py --config 4 --envs 2 --ctrl 1 > gpurun_out/${TAG}_racecheck.log 2>&1; echo "EXIT $?" >> gpurun_out/${TAG}_racecheck.log
timeout 900 compute-sanitizer --tool memcheck python tools/prof_rollout.py --config 4 --envs 2 --ctrl 1 > gpurun_out/${TAG}_memcheck.log 2>&1; echo "EXIT $?" >> gpurun_out/${TAG}_memcheck.log
timeout 900 compute-sanitizer --tool synccheck python tools/prof_rollout.py --config 3 --envs 2 --ctrl 1 > gpurun_out/${TAG}_synccheck.log 2>&1; echo "EXIT $?" >> gpurun_out/${TAG}_synccheck.log
fi
du -sh gpurun_out
