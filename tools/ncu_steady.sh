#!/bin/bash
# Steady-state ncu --set full captures (cfg4, one control step) of the hot
# kernels: forward p2g/g2p from substep ~16, adjoint g2p_adj/p2g_adj from the
# middle of the backward pass.  usage: bash tools/ncu_steady.sh TAG [envs] [fwd-regex] [adj-regex]
TAG=${1:-steady}
ENVS=${2:-1024}
FRE=${3:-"^k_(p2g|g2p)$"}
ARE=${4:-"^k_(g2p_adj|p2g_adj)$"}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$FRE" --launch-skip 32 --launch-count 2 \
  -o gpurun_out/${TAG}_fwd -f python tools/prof_rollout.py --config 4 --envs $ENVS --ctrl 1 > gpurun_out/${TAG}_ncu_fwd.log 2>&1
echo "NCU fwd EXIT $?" >> gpurun_out/${TAG}_ncu_fwd.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$ARE" --launch-skip 20 --launch-count 2 \
  -o gpurun_out/${TAG}_adj -f python tools/prof_rollout.py --config 4 --envs $ENVS --ctrl 1 > gpurun_out/${TAG}_ncu_adj.log 2>&1
echo "NCU adj EXIT $?" >> gpurun_out/${TAG}_ncu_adj.log
ls -la gpurun_out
