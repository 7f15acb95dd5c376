#!/bin/bash
# build and run the sort micro-benchmark variants (dev tool)
set -e
mkdir -p build
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_1308_3203_b200/csrc"
$NV tools/sortbench.cu paper_1308_3203_b200/csrc/sort.cu -o build/sortbench
$NV -DSORT_PHASE_TIMING tools/sortbench.cu paper_1308_3203_b200/csrc/sort.cu -o build/sortbench_t
if [ -f build/sort_prev.cu ]; then
  cp build/sort_prev.cu paper_1308_3203_b200/csrc/_sort_prev.cu
  $NV tools/sortbench.cu paper_1308_3203_b200/csrc/_sort_prev.cu -o build/sortbench_prev 2>/dev/null || true
  rm -f paper_1308_3203_b200/csrc/_sort_prev.cu
fi
