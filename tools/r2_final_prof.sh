#!/bin/bash
# usage: gpurun -- bash tools/r2_final_prof.sh TAG
# ncu --set full of every tile kernel on cfg4 (1,024 envs) and of the SVD-law
# kernels on cfg3 (256 envs), plus the launch list (gpu__time_duration) of the
# default bench command: one whole rollout (the second warm-up step: launches
# 7,700 .. 15,399, forward + replay + adjoint).
TAG=${1:-f}
bash tools/r2_prof2.sh ${TAG}4 4 1024 2 k_bin k_cellsort k_p2g k_grid k_g2p k_g2p_adj k_grid_adj k_p2g_adj
bash tools/r2_prof2.sh ${TAG}3 3 256 1 k_p2g k_g2p k_g2p_adj k_p2g_adj
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 7700 -c 7700 --csv --log-file gpurun_out/${TAG}_bench_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_ncu.log 2>&1
du -sh gpurun_out
