#!/bin/bash
# build the sort micro-benchmark variants (dev tool); extra -D flags via $SB_FLAGS
set -e
mkdir -p build
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -lineinfo -Iinclude -Ipaper_1308_3203_b200/csrc"
$NV $SB_FLAGS tools/sortbench.cu paper_1308_3203_b200/csrc/sort.cu -o build/sortbench
$NV $SB_FLAGS -DSORT_PHASE_TIMING tools/sortbench.cu paper_1308_3203_b200/csrc/sort.cu -o build/sortbench_t
