for v in default gadj5; do
  if [ $v == gadj5 ]; then export DIFFMPM_SO=variants/lib_gadj5.so; else unset DIFFMPM_SO; fi
  timeout 600 python bench.py --config 3 --ctrl 4 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vc_${v}_cfg3.json 2>/dev/null
  timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vc_${v}_cfg2.json 2>/dev/null
  timeout 300 python bench.py --envs 128 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/vc_${v}_e128.json 2>/dev/null
done
