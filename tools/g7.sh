timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/t7.log 2>&1; echo EXIT $? >> gpurun_out/t7.log
timeout 600 python bench.py --config 3 --ctrl 2 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/b2_cfg3.json 2> gpurun_out/b2_cfg3.err
timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b2_cfg1.json 2> gpurun_out/b2_cfg1.err
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_grid_adj" -s 4 -c 1 -o gpurun_out/ga_new -f python tools/prof_rollout.py --config 4 --envs 1024 --ctrl 2 > gpurun_out/ga_ncu.log 2>&1
