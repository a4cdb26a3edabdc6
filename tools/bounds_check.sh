#!/bin/bash
# usage: gpurun -- bash tools/bounds_check.sh TAG
# The GPU suite against a bounds-checked build (-DDM_DEBUG_BOUNDS: DM_CHECK in
# the state / perm / block / node indexing traps on a violation), in both
# scheduling modes -- the stand-in for compute-sanitizer, which this pool does
# not allow.  The library is built here by tools/build_debug.sh.
TAG=${1:-bc}
mkdir -p gpurun_out
for co in 0 1; do
  DIFFMPM_SO=paper_2412_12089_b200/libdiffmpm_dbg.so DIFFMPM_COOP=$co DIFFMPM_GRID_COOP=$co timeout 1500 \
    python -m pytest tests -m gpu -q > gpurun_out/${TAG}_coop${co}.log 2>&1
  echo "EXIT $?" >> gpurun_out/${TAG}_coop${co}.log
done
