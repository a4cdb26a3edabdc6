#!/bin/bash
# round-2 baseline: GPU tests + small-config benches (kernel-class split)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2b_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/r2b_tests.log
for c in 1 2; do
timeout 600 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2b_cfg$c.json 2> gpurun_out/r2b_cfg$c.err
done
timeout 600 python bench.py --config 4 --envs 128 --steps 3 --warmup 2 --no-cpu-baseline --no-e2e > gpurun_out/r2b_cfg4_128.json 2> gpurun_out/r2b_cfg4_128.err
