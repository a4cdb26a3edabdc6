#!/bin/bash
# Steady-state ncu --set full capture of every kernel class of the cfg4
# substep (one launch each) + the launch list of a short bench run.
# usage: bash tools/ncu_all.sh TAG
TAG=${1:-all}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(bin|cellsort|p2g|grid|g2p)$" \
  --launch-skip 80 --launch-count 5 -o gpurun_out/${TAG}_fwd -f \
  python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 1 > gpurun_out/${TAG}_ncu_fwd.log 2>&1
echo "fwd EXIT $?" >> gpurun_out/${TAG}_ncu_fwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_(g2p_adj|grid_adj|p2g_adj|env_reduce)$" \
  --launch-skip 40 --launch-count 4 -o gpurun_out/${TAG}_adj -f \
  python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 1 > gpurun_out/${TAG}_ncu_adj.log 2>&1
echo "adj EXIT $?" >> gpurun_out/${TAG}_ncu_adj.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --ctrl 2 --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_launches.log 2>&1
echo "launches EXIT $?" >> gpurun_out/${TAG}_launches.log
