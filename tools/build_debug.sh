#!/bin/bash
# paper_2412_12089_b200/libdiffmpm_dbg.so: the library with DM_DEBUG_BOUNDS checks (tools/bounds_check.sh)
cd "$(dirname "$0")/.."
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --shared -Xcompiler -fPIC -DDM_DEBUG_BOUNDS \
  -o paper_2412_12089_b200/libdiffmpm_dbg.so paper_2412_12089_b200/csrc/dm_context.cu
