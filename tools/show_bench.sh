#!/bin/bash
# usage: bash tools/show_bench.sh TAG : test/smoke verdicts and bench lines of a gpurun tag
TAG=$1
tail -2 gpurun_out/${TAG}_tests.log; tail -2 gpurun_out/${TAG}_smoke.log
for f in gpurun_out/${TAG}_cfg*.json; do
  python -c "import json;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f',round(d['value']/1e9,4),'e9',round(d['ms_per_step'],2),'ms',{k:round(v,2) for k,v in d.get('kernel_ms_per_step',{}).items()})" 2>&1 | tail -1
done
