#!/bin/bash
# usage: gpurun -- bash tools/gpu_tests.sh TAG [pytest selection args...]
TAG=${1:-t}; shift
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x "$@" > gpurun_out/${TAG}_tests.log 2>&1; echo "TESTS EXIT $?" >> gpurun_out/${TAG}_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "SMOKE EXIT $?" >> gpurun_out/${TAG}_smoke.log
