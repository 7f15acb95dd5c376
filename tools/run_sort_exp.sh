#!/bin/bash
# sort micro-benchmark on the GPU box (dev tool)
./tools/sortbench.sh > gpurun_out/sb_build.log 2>&1 || { cat gpurun_out/sb_build.log; exit 1; }
for v in 1 0; do for pat in stencil random; do echo "== variant $v $pat"; ./build/sortbench 29360128 24 $pat 10 $v | grep -v variant; done; done
for v in 1 0; do echo "== phase timing variant $v (stencil)"; ./build/sortbench_t 29360128 24 stencil 5 $v | grep -v variant; done
