mkdir -p gpurun_out
for v in base cg2; do
  if [ $v == cg2 ]; then export DIFFMPM_SO=paper_2412_12089_b200/libdiffmpm_cg2.so; else unset DIFFMPM_SO; fi
  timeout 300 python bench.py --envs 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cg_${v}_e128.json 2>/dev/null
  timeout 300 python bench.py --envs 256 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cg_${v}_e256.json 2>/dev/null
  timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cg_${v}_cfg2.json 2>/dev/null
  timeout 300 python bench.py --config 1 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/cg_${v}_cfg1.json 2>/dev/null
done
DIFFMPM_SO=paper_2412_12089_b200/libdiffmpm_cg2.so timeout 900 python -m pytest tests -m gpu -q -x -k "parity or modes or sort" > gpurun_out/cg2_tests.log 2>&1; echo EXIT $? >> gpurun_out/cg2_tests.log
