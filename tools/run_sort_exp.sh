#!/bin/bash
# sort micro-benchmark experiments on the GPU box (dev tool)
N=${SB_N:-7340032}
for cfg in ""; do
  SB_FLAGS="$cfg" ./tools/sortbench.sh > gpurun_out/sb_build.log 2>&1 || { cat gpurun_out/sb_build.log; exit 1; }
  for pat in stencil random; do for v in 1 0; do echo "== [$cfg] $pat variant $v"; ./build/sortbench $N 24 $pat 10 $v | grep -E "median|verify"; done; done
  echo "== [$cfg] phases (persistent)"; ./build/sortbench_t $N 24 stencil 5 1 | grep phase
done
