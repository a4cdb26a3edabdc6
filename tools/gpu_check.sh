#!/bin/bash
# One gpurun call: GPU tests, smoke, bench (cfg4 default), ncu --set full of the hot kernels.
# usage: gpurun -- bash tools/gpu_check.sh [tag] [skip-tests]
TAG=${1:-run}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
if [ "$2" != "skip-tests" ]; then
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_gpu_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/${TAG}_gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "SMOKE EXIT $?" >> gpurun_out/${TAG}_smoke.log
fi
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "BENCH EXIT $?" >> gpurun_out/${TAG}_bench.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(p2g|g2p)" -c 2 -o gpurun_out/${TAG}_fwd -f python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 1 > gpurun_out/${TAG}_ncu_fwd.log 2>&1; echo "NCU EXIT $?" >> gpurun_out/${TAG}_ncu_fwd.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_(g2p|p2g)_adj" -c 2 -o gpurun_out/${TAG}_adj -f python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 1 > gpurun_out/${TAG}_ncu_adj.log 2>&1; echo "NCU EXIT $?" >> gpurun_out/${TAG}_ncu_adj.log
